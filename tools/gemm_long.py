"""Sustained exhaustive-Pearson throughput (power-capped regime): 88 region pairs at n=1000 (a row of
the context matrix) repeated `reps` times, with nvidia-smi clocks sampled during the run.
Development tool; prints one JSON line."""
import json
import subprocess
import sys

import torch

sys.path.insert(0, ".")
from paper_2309_03308_b200 import binding as cb  # noqa: E402
from paper_2309_03308_b200 import synth  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
cfg = synth.C4
spec = synth.spec_of(cfg)
vals = synth.generate(spec, device="cuda")
f = cb.corr_field_create(vals, spec.nx, spec.ny, spec.nz, spec.members)
del vals
torch.cuda.empty_cache()
bricks = synth.bricks_of(cfg)
A, B = cb.boxes([bricks[5]] * 88), cb.boxes(bricks)
pairs = sum((a.x1 - a.x0) * (a.y1 - a.y0) * (a.z1 - a.z0) * (b.x1 - b.x0) * (b.y1 - b.y0) * (b.z1 - b.z0)
            for a, b in zip(A, B))
cb.corr_region_max(f, None, cb.CORR_PEARSON, 0, A, B, 0, 0)
torch.cuda.synchronize()
smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits",
                        "-lms", "100"], stdout=subprocess.PIPE, text=True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    cb.corr_region_max(f, None, cb.CORR_PEARSON, 0, A, B, 0, 0)
e1.record()
torch.cuda.synchronize()
smi.terminate()
lines = [l.split(",") for l in smi.communicate()[0].strip().splitlines() if "," in l]
clk = sorted(float(a) for a, _ in lines)
s = e0.elapsed_time(e1) / 1e3 / reps
tf = 6 * pairs * spec.members / s / 1e12
med = clk[len(clk) // 2] if clk else None
print(json.dumps({"s_per_row": s, "tc_tflops_3x": tf, "sm_mhz_median": med,
                  "tflops_per_ghz": tf / (med / 1e3) if med else None}))
