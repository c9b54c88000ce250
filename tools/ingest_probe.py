"""Field ingest cost breakdown at C4 (development tool): pinned H2D copy, corr_field_create from a
device buffer, from pinned host memory, and destroy."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2309_03308_b200 import binding as cb  # noqa: E402
from paper_2309_03308_b200 import synth  # noqa: E402

spec = synth.spec_of(synth.C4)
vals = synth.generate(spec, device="cuda")
host = torch.empty_like(vals, device="cpu").pin_memory()
host.copy_(vals)
torch.cuda.synchronize()
res = {}
for rep in range(2):
    t = time.perf_counter()
    vals.copy_(host, non_blocking=True)
    torch.cuda.synchronize()
    res["h2d_s"] = time.perf_counter() - t
    t = time.perf_counter()
    f = cb.corr_field_create(vals, spec.nx, spec.ny, spec.nz, spec.members)
    res["create_from_device_s"] = time.perf_counter() - t
    t = time.perf_counter()
    f.close()
    res["destroy_s"] = time.perf_counter() - t
    t = time.perf_counter()
    f = cb.corr_field_create(host, spec.nx, spec.ny, spec.nz, spec.members, device=0)
    res["create_from_pinned_host_s"] = time.perf_counter() - t
    f.close()
# in-place re-ingest (corr_field_update: transpose, fp64 stats, tf32 split, per-row sort), CUDA events
f = cb.corr_field_create(vals, spec.nx, spec.ny, spec.nz, spec.members)
cb.corr_field_update(f, vals)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    cb.corr_field_update(f, vals)
e1.record()
torch.cuda.synchronize()
res["update_device_ms"] = e0.elapsed_time(e1) / 3
f.close()
print(json.dumps(res))
