"""C3 (n = 100): KSG region max with the warp kernel, sweep vs CORR_F_KSG_DENSE (development tool)."""
import sys, json, torch
sys.path.insert(0, ".")
from paper_2309_03308_b200 import binding as cb
from paper_2309_03308_b200 import synth
spec = synth.spec_of(synth.C3)
vals = synth.generate(spec, device="cuda")
f = cb.corr_field_create(vals, spec.nx, spec.ny, spec.nz, spec.members)
A, B = synth.context_pairs(synth.bricks_of(synth.C3))
A, B = cb.boxes(A), cb.boxes(B)
for name, meas in (("sweep", cb.CORR_KSG), ("dense", cb.CORR_KSG | cb.CORR_F_KSG_DENSE)):
    m0, _ = cb.corr_region_max(f, None, meas, 3, A, B, 4096, 1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        m, a = cb.corr_region_max(f, None, meas, 3, A, B, 4096, 1)
    e1.record(); torch.cuda.synchronize()
    s = e0.elapsed_time(e1) / 3 / 1e3
    print(name, round(len(A) * 4096 / s / 1e6, 1), "Mpairs/s", float(m.max()), bool(torch.equal(m, m0)))
