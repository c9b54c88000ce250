"""Diagnostic: what makes the KSG kernel faster when something runs concurrently (dev tool)."""
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
dev2 = torch.empty_like(vals)
A, B = synth.context_pairs(synth.bricks_of(synth.C4))
A, B = cb.boxes(A), cb.boxes(B)
S = 1024
side = torch.cuda.Stream()
big = torch.empty(1 << 28, device="cuda")


def timed(concurrent=None):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    if concurrent is not None:
        with torch.cuda.stream(side):
            concurrent()
    cb.corr_region_max(f, None, cb.CORR_KSG, 3, A, B, S, 20230907)
    e1.record()
    torch.cuda.synchronize()
    return round(e0.elapsed_time(e1), 2)


res = {"alone": [timed() for _ in range(2)]}
res["h2d_copy_only"] = timed(lambda: dev2.copy_(host, non_blocking=True))
res["tiny_kernel_first"] = timed(lambda: big[:1024].add_(1.0))
res["memset_kernels"] = timed(lambda: [big.add_(1.0) for _ in range(20)])
res["alone_again"] = timed()
print(json.dumps(res))
