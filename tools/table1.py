"""Table 1 shape of the paper: one reference point vs all 1.76 M grid points,
n = 100 and 1000, PPMCC and KMI (k = 3 and the paper's k = ceil(3n/100)).  Development tool:
prints one JSON line with GPU seconds per one-to-all sweep (CUDA events)."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2309_03308_b200 import binding as cb  # noqa: E402
from paper_2309_03308_b200 import synth  # noqa: E402


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3


res = {"paper_rtx3090_s": {"ppmcc_100": 0.002, "kmi_100": 0.672, "ppmcc_1000": 0.21, "kmi_1000": 35.9}}
for cfg in (synth.C3, synth.C4):
    spec = synth.spec_of(cfg)
    vals = synth.generate(spec, device="cuda")
    f = cb.corr_field_create(vals, spec.nx, spec.ny, spec.nz, spec.members)
    del vals
    torch.cuda.empty_cache()
    P = spec.points
    ref = (10 * spec.ny + 176) * spec.nx + 125  # a grid point in the middle of the domain
    ia = torch.full((P,), ref, dtype=torch.int64, device="cuda")
    ib = torch.arange(P, dtype=torch.int64, device="cuda")
    out = torch.empty(P, dtype=torch.float32, device="cuda")
    n = spec.members
    kp = max(1, -(-3 * n // 100))
    res[f"ppmcc_{n}"] = timed(lambda: cb.corr_eval_pairs(f, None, cb.CORR_PEARSON, 0, ia, ib, out))
    res[f"kmi_{n}_k3"] = timed(lambda: cb.corr_eval_pairs(f, None, cb.CORR_KSG, 3, ia, ib, out), reps=1)
    res[f"kmi_{n}_k{kp}"] = timed(lambda: cb.corr_eval_pairs(f, None, cb.CORR_KSG, 0, ia, ib, out), reps=1)
    print(json.dumps(res), flush=True)
    f.close()
