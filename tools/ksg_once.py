"""Runs one KSG region-max launch on the C4 field (ncu target; development tool)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2309_03308_b200 import binding as cb  # noqa: E402
from paper_2309_03308_b200 import synth  # noqa: E402

cfg = {"c3": synth.C3, "c4": synth.C4}[sys.argv[1] if len(sys.argv) > 1 else "c4"]
S = int(sys.argv[2]) if len(sys.argv) > 2 else 16
spec = synth.spec_of(cfg)
vals = synth.generate(spec, device="cuda")
f = cb.corr_field_create(vals, spec.nx, spec.ny, spec.nz, spec.members)
del vals
A, B = synth.context_pairs(synth.bricks_of(cfg))
for _ in range(2):
    m, a = cb.corr_region_max(f, None, cb.CORR_KSG, 3, A, B, S, 1)
torch.cuda.synchronize()
print("ok", float(m[0]))
