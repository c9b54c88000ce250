"""Config 5 (BASELINE.json configs[4]): two fields on 250x352x20, n = 1000, the full 88 x 88 ordered
inter-variable region matrix: exhaustive Pearson maxima over all 3.1e12 point
pairs (tcgen05 path) and KSG maxima over 1024 sampled pairs per region pair.  Development tool;
prints one JSON line with wall times and throughputs."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2309_03308_b200 import binding as cb  # noqa: E402
from paper_2309_03308_b200 import synth  # noqa: E402

cfg = synth.C5
fields = []
for var in (1, 2):
    spec = synth.spec_of(cfg, var)
    vals = synth.generate(spec, device="cuda")
    fields.append(cb.corr_field_create(vals, spec.nx, spec.ny, spec.nz, spec.members))
    del vals
    torch.cuda.empty_cache()
fa, fb = fields
A, B = synth.matrix_pairs(synth.bricks_of(cfg))
pairs = sum(synth.box_size(a) * synth.box_size(b) for a, b in zip(A, B))
A, B = cb.boxes(A), cb.boxes(B)
res = {"region_pairs": len(A), "point_pairs": pairs}
for name, measure, S in (("ksg_S1024", cb.CORR_KSG, 1024), ("pearson_exhaustive", cb.CORR_PEARSON, 0)):
    torch.cuda.synchronize()
    cb.corr_gemm_flops(0, reset=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t = time.time()
    e0.record()
    m, a = cb.corr_region_max(fa, fb, measure, 3, A, B, S, 5)
    e1.record()
    torch.cuda.synchronize()
    s = e0.elapsed_time(e1) / 1e3
    n_pairs = len(A) * S if S else pairs
    res[name] = {"s": s, "wall_s": time.time() - t, "pairs_per_s": n_pairs / s,
                 "max": float(m.max()), "nan": int(torch.isnan(m).sum())}
    if S == 0:
        res[name]["logical_tflops"] = 2 * pairs * 1000 / s / 1e12
        res[name]["dense_equivalent_tc_tflops_3x"] = 6 * pairs * 1000 / s / 1e12
        res[name]["executed_tc_tflops"] = sum(cb.corr_gemm_flops(0, reset=True)) / s / 1e12
    print(json.dumps(res), flush=True)
