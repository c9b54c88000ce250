"""Quick throughput probe of the hot path on one GPU (development tool, not the bench)."""
import json
import sys
import time

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


def main():
    which = sys.argv[1:] or ["c3", "c4"]
    res = {}
    for name in which:
        cfg = {"c3": synth.C3, "c4": synth.C4}[name]
        spec = synth.spec_of(cfg)
        t = time.time()
        vals = synth.generate(spec, device="cuda")
        torch.cuda.synchronize()
        res[name + "_gen_s"] = time.time() - t
        t = time.time()
        f = cb.corr_field_create(vals, spec.nx, spec.ny, spec.nz, spec.members)
        res[name + "_create_s"] = time.time() - t
        del vals
        torch.cuda.empty_cache()
        A, B = synth.context_pairs(synth.bricks_of(cfg))
        A, B = cb.boxes(A), cb.boxes(B)
        for S in ((64, 1024) if name == "c3" else (16, 64)):
            dt = timed(lambda: cb.corr_region_max(f, None, cb.CORR_KSG, 3, A, B, S, 1), reps=2)
            pairs = len(A) * S
            n = spec.members
            res[f"{name}_ksg_S{S}"] = {"s": dt, "pairs_per_s": pairs / dt, "cmp_per_s": pairs * n * (n - 1) / dt}
            dt = timed(lambda: cb.corr_region_max(f, None, cb.CORR_PEARSON, 0, A, B, S * 16, 1), reps=2)
            res[f"{name}_pearson_S{S * 16}"] = {"s": dt, "pairs_per_s": len(A) * S * 16 / dt}
        print(json.dumps(res), flush=True)
        f.close()
    print(json.dumps(res))


if __name__ == "__main__":
    main()
