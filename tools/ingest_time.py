"""Times corr_field_update from a device buffer at C4 (transpose + stats + sort; development tool)."""
import json
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2309_03308_b200 import binding as cb  # noqa: E402
from paper_2309_03308_b200 import synth  # noqa: E402

spec = synth.spec_of(synth.C4)
vals = synth.generate(spec, device="cuda")
f = cb.corr_field_create(vals, spec.nx, spec.ny, spec.nz, spec.members)
for _ in range(2):
    cb.corr_field_update(f, vals)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    cb.corr_field_update(f, vals)
e1.record()
torch.cuda.synchronize()
cb.corr_check(f)
print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("CORR_")},
                  "update_ms": e0.elapsed_time(e1) / 5}))
