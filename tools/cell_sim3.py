"""Cell k-NN cost model, variant 'task waves' (development tool, round 2).

Own column: warp per column, lockstep up/down scan (lane = member, y order).  Then waves
(L1, R1, L2, R2, ...): a wave's tasks are the members whose column at that side/depth is still
needed (x-gap < l[k-1], side not ended); tasks are compacted and processed 32 per warp group,
lane = task (member state loaded from shared memory); group cost = SETUP + max steps * STEP.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from sweep_sim import pairs_of, warp_cost  # noqa: E402
from cell_sim2 import lane_scan, K  # noqa: E402


def pair_cost(x, y, C, STEP, SETUP, OWN0, order="member"):
    n = len(x)
    ncol = (n + C - 1) // C
    yr = np.empty(n, np.int64)
    yr[np.argsort(y, kind="stable")] = np.arange(n)
    cols = [np.arange(c * C, min(n, (c + 1) * C))[np.argsort(yr[c * C:min(n, (c + 1) * C)], kind="stable")]
            for c in range(ncol)]
    colof = np.arange(n) // C
    L = {}
    cost = 0.0
    st = dict(own=0, groups=0, gsteps=0, tasks=0, cands=0, waves=0)
    for w in range(ncol):
        mem = cols[w]
        cx, cy = x[mem], y[mem]
        ms = 0
        for l_, i in enumerate(mem):
            l, s, cc = lane_scan([np.inf] * K, x[i], y[i], cx, cy, l_ + 1, l_ - 1)
            L[i] = l
            ms = max(ms, s)
            st['cands'] += cc
        cost += OWN0 + ms * STEP
        st['own'] += ms
    alive = {0: np.ones(n, bool), 1: np.ones(n, bool)}
    depth = 1
    while alive[0].any() or alive[1].any():
        for side in (0, 1):
            tasks = []
            for i in np.where(alive[side])[0]:
                c = colof[i] - depth if side == 0 else colof[i] + depth
                if c < 0 or c >= ncol:
                    alive[side][i] = False
                    continue
                gap = np.float32(x[i] - x[(c + 1) * C - 1]) if side == 0 else np.float32(x[c * C] - x[i])
                if gap < L[i][K - 1]:
                    tasks.append((i, c))
                else:
                    alive[side][i] = False
            st['waves'] += 1
            cost += SETUP * ((n + 127) // 128)  # the wave's gap tests + compaction over all members
            res = []
            for i, c in tasks:
                cm = cols[c]
                start = int(np.sum(yr[cm] < (yr[i] // 32) * 32))
                l, s, cc = lane_scan(L[i], x[i], y[i], x[cm], y[cm], start, start - 1)
                L[i] = l
                res.append(s)
                st['cands'] += cc
            st['tasks'] += len(tasks)
            if order == "sorted":
                res = sorted(res)
            for g in range(0, len(res), 32):
                ms = max(res[g:g + 32])
                cost += SETUP + ms * STEP
                st['groups'] += 1
                st['gsteps'] += ms
        depth += 1
    eps = np.array([L[i][K - 1] for i in range(n)], np.float32)
    return cost, eps, st


def main(npairs=4, STEP=18.0, SETUP=20.0, OWN0=10.0):
    tc, told = 0.0, 0.0
    agg = {}
    for xa, xb in pairs_of(npairs):
        if xb.std() > xa.std():
            xa, xb = xb, xa
        o = np.argsort(xa, kind="stable")
        x, y = xa[o], xb[o]
        n = len(x)
        d = np.maximum(np.abs(x[:, None] - x[None, :]), np.abs(y[:, None] - y[None, :]))
        np.fill_diagonal(d, np.inf)
        eps = np.partition(d, K - 1, 1)[:, K - 1]
        c, e, st = pair_cost(x, y, 32, STEP, SETUP, OWN0)
        assert np.array_equal(e, eps)
        for k_, v in st.items():
            agg[k_] = agg.get(k_, 0) + v
        old = sum(warp_cost(x, y, b0, 32, 1, 32, False)[0] for b0 in range(0, n, 32))
        tc += c
        told += old
    print({k_: v / npairs for k_, v in agg.items()})
    print(f"waves model {tc / npairs:.0f} warp-ALU per pair vs sweep model {told / npairs:.0f} ({told / tc:.2f}x)")


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
