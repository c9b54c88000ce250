"""Config 2 (BASELINE.json configs[1]): the focus view of one region pair -- two 32x32x20 bricks of
the C3-shaped field (n = 100), ALL 4.19e8 point pairs: exhaustive Pearson block (tcgen05 path) and
exhaustive KSG MI k = 3, each reduced to the pair's max/argmax, plus
the focus refinement into (M/2)^2 sub-brick pairs (NEXT #3, synth.refine) in one call.
Development tool; prints one JSON line (CUDA-event seconds)."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2309_03308_b200 import binding as cb  # noqa: E402
from paper_2309_03308_b200 import synth  # noqa: E402


def timed(fn):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1e3, out


cfg = synth.C2
spec = synth.spec_of(cfg)
vals = synth.generate(spec, device="cuda")
f = cb.corr_field_create(vals, spec.nx, spec.ny, spec.nz, spec.members)
del vals
A, B = synth.C2_REGION_A, synth.C2_REGION_B
npairs = synth.box_size(A) * synth.box_size(B)
res = {"config": "C2 focus: bricks %s x %s, n=%d" % (A, B, spec.members), "point_pairs": npairs}
for name, measure in (("pearson_block", cb.CORR_PEARSON), ("ksg_k3", cb.CORR_KSG)):
    s, (m, a) = timed(lambda: cb.corr_region_max(f, None, measure, 3, cb.boxes([A]), cb.boxes([B]), 0, 0))
    res[name] = {"s": s, "pairs_per_s": npairs / s, "max": float(m[0]), "argmax": [int(a[0][0]), int(a[0][1])]}
# focus refinement: children of both bricks, all (M/2)^2 child pairs, exhaustive, in one call
ca, cbx = synth.refine(A, 8), synth.refine(B, 8)
RA = [x for x in ca for _ in cbx]
RB = [y for _ in ca for y in cbx]
for name, measure in (("refine_pearson", cb.CORR_PEARSON), ("refine_ksg_k3", cb.CORR_KSG)):
    s, (m, a) = timed(lambda: cb.corr_region_max(f, None, measure, 3, cb.boxes(RA), cb.boxes(RB), 0, 0))
    res[name] = {"s": s, "child_pairs": len(RA), "pairs_per_s": npairs / s, "matrix_max": float(m.max())}
print(json.dumps(res), flush=True)
