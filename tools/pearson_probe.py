"""Times the sampled Pearson region max of the bench (C4, 3828 region pairs x S = 4096) with CUDA
events (development tool): pairs/s and the assumed-bytes HBM rate."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2309_03308_b200 import binding as cb  # noqa: E402
from paper_2309_03308_b200 import synth  # noqa: E402

spec = synth.spec_of(synth.C4)
vals = synth.generate(spec, device="cuda")
f = cb.corr_field_create(vals, spec.nx, spec.ny, spec.nz, spec.members)
del vals
torch.cuda.empty_cache()
A, B = synth.context_pairs(synth.bricks_of(synth.C4))
A, B = cb.boxes(A), cb.boxes(B)
S = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
cb.corr_region_max(f, None, cb.CORR_PEARSON, 0, A, B, S, 20230907)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 5
e0.record()
for _ in range(reps):
    m, a = cb.corr_region_max(f, None, cb.CORR_PEARSON, 0, A, B, S, 20230907)
e1.record()
torch.cuda.synchronize()
s = e0.elapsed_time(e1) / reps / 1e3
pairs = len(A) * S
print(json.dumps({"ms": s * 1e3, "pairs_per_s": pairs / s, "assumed_GBps": pairs * (4 * spec.members + 8) / s / 1e9,
                  "max0": float(m[0])}))
