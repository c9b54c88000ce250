"""The bench's two Pearson calls on the C4 field (ncu target; development tool): the sampled
region max over all 3828 region pairs (S = 4096) and the exhaustive focus block (tcgen05 GEMM)."""
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
fa, fb = cb.boxes([synth.C2_REGION_A]), cb.boxes([synth.C2_REGION_B])
for _ in range(2):
    m1, a1 = cb.corr_region_max(f, None, cb.CORR_PEARSON, 0, A, B, 4096, 20230907)
    m2, a2 = cb.corr_region_max(f, None, cb.CORR_PEARSON, 0, fa, fb, 0, 0)
torch.cuda.synchronize()
print("ok", float(m1[0]), float(m2[0]))
