"""Latency of one BOS-shaped batch (the acquisitions of all brick pairs are batched and
sent to the GPU together): 3828 point pairs, one per region pair of the context view, KSG k=3 and
Pearson, through corr_eval_pairs -- plain stream launches and a captured CUDA graph.  Development
tool; prints one JSON line."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2309_03308_b200 import binding as cb  # noqa: E402
from paper_2309_03308_b200 import synth  # noqa: E402


def timed(fn, reps=50):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


res = {}
for cfg in (synth.C3, synth.C4):
    spec = synth.spec_of(cfg)
    vals = synth.generate(spec, device="cuda")
    f = cb.corr_field_create(vals, spec.nx, spec.ny, spec.nz, spec.members)
    del vals
    torch.cuda.empty_cache()
    a, b = synth.random_pairs(spec.points, 3828, seed=1)
    a, b = a.cuda(), b.cuda()
    out = torch.empty(3828, dtype=torch.float32, device="cuda")
    s = torch.cuda.Stream()
    for name, measure in (("ksg", cb.CORR_KSG), ("pearson", cb.CORR_PEARSON)):
        res[f"n{spec.members}_{name}_stream_ms"] = timed(lambda: cb.corr_eval_pairs(f, None, measure, 3, a, b, out))
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            cb.corr_eval_pairs(f, None, measure, 3, a, b, out, stream=s)
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=s):
                cb.corr_eval_pairs(f, None, measure, 3, a, b, out, stream=s)
        res[f"n{spec.members}_{name}_graph_ms"] = timed(g.replay)
    f.close()
print(json.dumps(res))
