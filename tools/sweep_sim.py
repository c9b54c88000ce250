"""SIMT cost model of the KSG sweep kernel (development tool; DESIGN.md §6 "Why the
executed-comparison fraction is capped").

Replays, on C4-shaped point pairs (n = 1000, k = 3, rows from the shared generator), the
warp-level schedule of ksg_sorted_kernel: a warp owns B x-consecutive members (R = 32/B lanes
per member, each lane taking every R-th candidate), scans its own block with the exact merge
network, then C-wide candidate chunks outward; the first chunk in each direction is exact, later
ones are filtered in groups of 4 (a group costs the merge network only if SOME lane's group
minimum beats its k-th distance); a direction stops once no lane's x-gap to the next chunk is
below its current k-th distance.  Costs are warp-ALU instructions: 5 per exactly merged value
(distance FMNMX + 4 min/max of the 2-value merge), 7 per filtered group of 4.
Every schedule is checked to reproduce the exact eps of brute force.

    python tools/sweep_sim.py [npairs]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2309_03308_b200 import synth  # noqa: E402

K, G = 3, 4
EXACT_V, FILT_G, SWEEP = 5.0, 7.0, 2.0


def pairs_of(npairs, seed=0):
    cfg = synth.C4
    spec = synth.spec_of(cfg)
    A, B = synth.context_pairs(synth.bricks_of(cfg))
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(npairs):
        r = int(rng.integers(len(A)))
        pts = []
        for box in (A[r], B[r]):
            x0, y0, z0, x1, y1, z1 = box
            x, y, z = rng.integers(x0, x1), rng.integers(y0, y1), rng.integers(z0, z1)
            pts.append(int((z * spec.ny + y) * spec.nx + x))
        out.append(tuple(pts))
    allp = sorted({p for ab in out for p in ab})
    rows = synth.rows(spec, torch.tensor(allp)).numpy()
    pos = {p: i for i, p in enumerate(allp)}
    return [(rows[pos[a]].astype(np.float32), rows[pos[b]].astype(np.float32)) for a, b in out]


def warp_cost(x, y, b0, Bk, R, C, share):
    n = len(x)
    mem = np.arange(b0, min(b0 + Bk, n))
    nm = len(mem)
    lm = np.repeat(mem, R)
    lr = np.tile(np.arange(R), nm)
    xi, yi = x[lm], y[lm]
    L = np.full((len(lm), K), np.inf)
    cost, cmps = 0.0, 0

    def dist(js):
        d = np.maximum(np.abs(xi[:, None] - x[None, js]), np.abs(yi[:, None] - y[None, js]))
        d[lm[:, None] == js[None, :]] = np.inf
        d[(js[None, :] % R) != lr[:, None]] = np.inf  # lane r takes every R-th candidate
        return d

    def insert(L, vals):
        return np.sort(np.concatenate([L, vals], 1), 1)[:, :K]

    js = np.arange(b0, min(b0 + Bk, n))
    L = insert(L, dist(js))
    cost += EXACT_V * len(js) / R
    cmps += len(js) * nm
    b1 = min(b0 + Bk, n)
    nlo, nhi = (b0 + C - 1) // C, (n - b1 + C - 1) // C
    state = {0: (0 if nlo else -1), 1: (0 if nhi else -1)}
    first = {0: True, 1: True}
    while state[0] >= 0 or state[1] >= 0:
        for dr in (0, 1):
            c = state[dr]
            if c < 0:
                continue
            js = np.arange(max(0, b0 - (c + 1) * C), b0 - c * C) if dr == 0 else np.arange(b1 + c * C, min(n, b1 + (c + 1) * C))
            t = L[:, K - 1].copy()
            if share and R > 1:
                t = t.reshape(nm, R).min(1).repeat(R)
            cost += SWEEP
            need = np.any(xi - x[js[-1]] < t) if dr == 0 else np.any(x[js[0]] - xi < t)
            if not need:
                state[dr] = -1
                continue
            d = dist(js)
            cmps += len(js) * nm
            if first[dr]:
                L = insert(L, d)
                cost += EXACT_V * len(js) / R
            else:
                order = np.arange(len(js))[::-1] if dr == 0 else np.arange(len(js))
                steps = len(js) // R
                own = [[ci for ci in order if js[ci] % R == lr[ln]] for ln in range(len(lm))]
                for g in range(0, steps, G):
                    vals = np.full((len(lm), G), np.inf)
                    for ln in range(len(lm)):
                        cols = own[ln][g:g + G]
                        vals[ln, :len(cols)] = d[ln, cols]
                    cost += FILT_G
                    if np.any(vals.min(1) < L[:, K - 1]):
                        cost += EXACT_V * G - G
                        L = insert(L, vals)
            first[dr] = False
            state[dr] = c + 1 if c + 1 < (nlo if dr == 0 else nhi) else -1
    cost += (R - 1) * 8  # combine a member's R partial lists
    return cost, cmps, np.sort(L.reshape(nm, R * K), 1)[:, K - 1]


def main(npairs=12):
    configs = [(32, 1, 32, False), (16, 2, 32, True), (16, 2, 16, True), (8, 4, 16, True)]
    tot = {c: [0.0, 0] for c in configs}
    for xa, xb in pairs_of(npairs):
        if xb.std() > xa.std():
            xa, xb = xb, xa
        o = np.argsort(xa, kind="stable")
        x, y = xa[o], xb[o]
        n = len(x)
        d = np.maximum(np.abs(x[:, None] - x[None, :]), np.abs(y[:, None] - y[None, :]))
        np.fill_diagonal(d, np.inf)
        eps = np.partition(d, K - 1, 1)[:, K - 1]
        strip = (np.abs(x[:, None] - x[None, :]) < eps[:, None]).sum(1) - 1
        tot.setdefault("strip", []).append(strip.mean())
        for c in configs:
            for b0 in range(0, n, c[0]):
                cw, cm, e = warp_cost(x, y, b0, *c)
                assert np.array_equal(e, eps[b0:b0 + c[0]])
                tot[c][0] += cw
                tot[c][1] += cm
    print(f"mean x-strip |dx| < eps: {np.mean(tot['strip']):.1f} members")
    for c in configs:
        B, R, C, share = c
        print(f"B={B:2d} lanes/member={R} chunk={C:2d}: warp-ALU per pair {tot[c][0] / npairs:8.0f}, "
              f"comparisons per member {tot[c][1] / npairs / 1000:6.1f}")


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 12)
