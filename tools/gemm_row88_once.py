"""One exhaustive Pearson row-88 call on the C4 field (brick 5 x all 88 bricks; ncu target,
development tool): the screened GEMM's per-kernel split."""
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
bricks = synth.bricks_of(synth.C4)
nrow = int(sys.argv[1]) if len(sys.argv) > 1 else 88
A, B = cb.boxes([bricks[5]] * nrow), cb.boxes(bricks[:nrow])
for _ in range(2):
    m, a = cb.corr_region_max(f, None, cb.CORR_PEARSON, 0, A, B, 0, 0)
torch.cuda.synchronize()
print("ok", float(m.max()))
