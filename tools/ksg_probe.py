"""KSG region-max throughput probe (development tool): pairs/s and executed comparisons/s."""
import json
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2309_03308_b200 import binding as cb  # noqa: E402
from paper_2309_03308_b200 import synth  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c4"
S = int(sys.argv[2]) if len(sys.argv) > 2 else 64
cfg = {"c3": synth.C3, "c4": synth.C4}[cfgname]
spec = synth.spec_of(cfg)
vals = synth.generate(spec, device="cuda")
f = cb.corr_field_create(vals, spec.nx, spec.ny, spec.nz, spec.members)
del vals
torch.cuda.empty_cache()
A, B = synth.context_pairs(synth.bricks_of(cfg))
A, B = cb.boxes(A), cb.boxes(B)
cb.corr_region_max(f, None, cb.CORR_KSG, 3, A, B, S, 1)
torch.cuda.synchronize()
cb.corr_ksg_comparisons(0, reset=True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 3
e0.record()
for _ in range(reps):
    m, a = cb.corr_region_max(f, None, cb.CORR_KSG, 3, A, B, S, 1)
e1.record()
torch.cuda.synchronize()
dt = e0.elapsed_time(e1) / reps / 1e3
cmp = cb.corr_ksg_comparisons(0, reset=True) / reps
if cmp == 0:  # the column-cell kernel counts only when asked (CORR_F_KSG_COUNT)
    cb.corr_region_max(f, None, cb.CORR_KSG | cb.CORR_F_KSG_COUNT, 3, A, B, S, 1)
    cmp = cb.corr_ksg_comparisons(0, reset=True)
n = spec.members
pairs = len(A) * S
peak = 148 * 128 * 1965e6 / 4
print(json.dumps({"cfg": cfgname, "S": S, "env": {k: v for k, v in os.environ.items() if k.startswith("CORR_")},
                  "s": dt, "pairs_per_s": pairs / dt, "dense_cmp_per_s": pairs * n * (n - 1) / dt,
                  "executed_cmp_per_s": cmp / dt, "executed_frac_of_dense": cmp / (pairs * n * (n - 1)),
                  "frac_executed_vs_peak": cmp / dt / peak, "max0": float(m[0])}))
