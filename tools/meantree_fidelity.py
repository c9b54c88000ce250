"""Mean-tree fidelity on synthetic data (the paper's Fig. 8 experiment):
region-pair maxima computed on the initial data (f=1) vs on 2x2x2 (f=2) and 4x4x4 (f=4) means,
for random brick pairs of 32x32x20.  The paper reports average deviations of 1.6 % / 1.7 % on
"Necker" with BOS@100; here the maxima are the exhaustive Pearson maximum (tcgen05 path) and the
KSG maximum over 100 random samples.  Prints one JSON line (development tool)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2309_03308_b200 import binding as cb  # noqa: E402
from paper_2309_03308_b200 import synth  # noqa: E402

cfg = synth.C3 if len(sys.argv) < 2 else {"c3": synth.C3, "c4": synth.C4}[sys.argv[1]]
npairs = 1000
spec = synth.spec_of(cfg)
vals = synth.generate(spec, device="cuda")
f1 = cb.corr_field_create(vals, spec.nx, spec.ny, spec.nz, spec.members)
del vals
torch.cuda.empty_cache()
bricks = synth.bricks_of(cfg)
rng = np.random.default_rng(7)
idx = [tuple(sorted(rng.choice(len(bricks), 2, replace=False))) for _ in range(npairs)]
out = {"config": cfg.name, "brick_pairs": npairs}
base = {}
for fac in (1, 2, 4):
    f = f1 if fac == 1 else cb.corr_field_aggregate(f1, fac, fac, fac)

    def sc(b):
        return (b[0] // fac, b[1] // fac, b[2] // fac, -(-b[3] // fac), -(-b[4] // fac), -(-b[5] // fac))

    A = [sc(bricks[i]) for i, _ in idx]
    B = [sc(bricks[j]) for _, j in idx]
    for name, measure, S in (("pearson_exhaustive", cb.CORR_PEARSON, 0), ("ksg_S100", cb.CORR_KSG, 100)):
        m, _ = cb.corr_region_max(f, None, measure, 3, A, B, S, 11)
        m = m.cpu().numpy().astype(np.float64)
        if fac == 1:
            base[name] = m
        else:
            rel = np.abs(m - base[name]) / np.maximum(np.abs(base[name]), 1e-12)
            out[f"{name}_f{fac}_mean_rel_dev"] = float(np.nanmean(rel))
            out[f"{name}_f{fac}_mean_abs_dev"] = float(np.nanmean(np.abs(m - base[name])))
    if fac != 1:
        f.close()
print(json.dumps(out))
