"""Throughput of the exhaustive Pearson block path (tcgen05 split-TF32 GEMM), development tool."""
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


res = {}
for cfg in (synth.C2, synth.C4):
    spec = synth.spec_of(cfg)
    vals = synth.generate(spec, device="cuda")
    f = cb.corr_field_create(vals, spec.nx, spec.ny, spec.nz, spec.members)
    del vals
    torch.cuda.empty_cache()
    n = spec.members
    bricks = synth.bricks_of(cfg)
    for name, A, B in (("focus", [synth.C2_REGION_A], [synth.C2_REGION_B]),
                       ("row88", [bricks[5]] * 88, bricks)):
        A, B = cb.boxes(A), cb.boxes(B)
        cb.corr_gemm_flops(0, reset=True)
        dt = timed(lambda: cb.corr_region_max(f, None, cb.CORR_PEARSON, 0, A, B, 0, 0))
        exe = sum(cb.corr_gemm_flops(0, reset=True)) / 4  # timed() runs the call 1 + 3 times
        pairs = sum((b.x1 - b.x0) * (b.y1 - b.y0) * (b.z1 - b.z0) * (a.x1 - a.x0) * (a.y1 - a.y0) * (a.z1 - a.z0)
                    for a, b in zip(A, B))
        res[f"{cfg.name}_{name}"] = {"s": dt, "pairs_per_s": pairs / dt,
                                    "logical_tflops": 2 * pairs * n / dt / 1e12,
                                    "dense_equivalent_tc_tflops_3x": 6 * pairs * n / dt / 1e12,
                                    "executed_tc_tflops": exe / dt / 1e12}
        print(json.dumps(res), flush=True)
    f.close()
