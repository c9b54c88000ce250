"""Diagnostic: KSG region-max time on a field after different update paths (development tool)."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2309_03308_b200 import binding as cb  # noqa: E402
from paper_2309_03308_b200 import synth  # noqa: E402

spec = synth.spec_of(synth.C4)
vals = synth.generate(spec, device="cuda")
f = cb.corr_field_create(vals, spec.nx, spec.ny, spec.nz, spec.members)
host = torch.empty((spec.members, spec.points), dtype=torch.float32, pin_memory=True)
host.copy_(vals)
A, B = synth.context_pairs(synth.bricks_of(synth.C4))
A, B = cb.boxes(A), cb.boxes(B)
S = 1024


def t_ksg():
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    cb.corr_region_max(f, None, cb.CORR_KSG, 3, A, B, S, 20230907)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


res = {}
t_ksg()
res["after_create_dev"] = [t_ksg() for _ in range(3)]
cb.corr_field_update(f, vals)
res["after_update_dev"] = [t_ksg() for _ in range(3)]
cb.corr_field_update(f, host.data_ptr())
res["after_update_host"] = [t_ksg() for _ in range(3)]
up = torch.cuda.Stream()
g = cb.corr_field_create(vals, spec.nx, spec.ny, spec.nz, spec.members)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
with torch.cuda.stream(up):
    cb.corr_field_update(g, host.data_ptr(), stream=up)
cb.corr_region_max(f, None, cb.CORR_KSG, 3, A, B, S, 20230907)
e1.record()
torch.cuda.synchronize()
res["ksg_overlapped_with_host_update"] = e0.elapsed_time(e1)
res["after_overlap"] = [t_ksg() for _ in range(2)]
print(json.dumps(res))
