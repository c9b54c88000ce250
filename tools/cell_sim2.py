"""Cell k-NN cost model, variant 'per-lane rounds' (development tool, round 2).

Columns of C = 32 x-consecutive members, y order inside a column; a warp owns a column (lane =
member).  Phase 1: own column, lockstep up/down scan.  Phase 2: rounds; in round r every lane
visits ITS next needed neighbour column (nearest first, alternating sides, a side ends at the
first column whose x-gap >= l[k-1]); the scan starts at the cell of the member's y band
(cellstart table, no search).  A round costs SETUP + (max steps over its lanes) * STEP.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from sweep_sim import pairs_of, warp_cost  # noqa: E402

K = 3


def ins(l, d):
    return sorted(l + [d])[:K]


def lane_scan(l, xi, yi, cx, cy, up, dn):
    """Scan one column (arrays cx, cy in y order) from up / dn pointers; returns l, steps, cands."""
    steps = cands = 0
    up_on, dn_on = up < len(cy), dn >= 0
    while up_on or dn_on:
        steps += 1
        if up_on:
            d = max(abs(np.float32(xi - cx[up])), abs(np.float32(yi - cy[up])))
            l = ins(l, d)
            cands += 1
            stop = np.float32(cy[up] - yi) >= l[K - 1]
            up += 1
            up_on = (not stop) and up < len(cy)
        if dn_on:
            d = max(abs(np.float32(xi - cx[dn])), abs(np.float32(yi - cy[dn])))
            l = ins(l, d)
            cands += 1
            stop = np.float32(yi - cy[dn]) >= l[K - 1]
            dn -= 1
            dn_on = (not stop) and dn >= 0
    return l, steps, cands


def pair_cost(x, y, C, STEP, SETUP, OWN0):
    n = len(x)
    ncol = (n + C - 1) // C
    yr = np.empty(n, np.int64)
    yr[np.argsort(y, kind="stable")] = np.arange(n)
    cols = []
    for c in range(ncol):
        t = np.arange(c * C, min(n, (c + 1) * C))
        cols.append(t[np.argsort(yr[t], kind="stable")])
    cost = 0.0
    eps = np.empty(n, np.float32)
    st = dict(own=0, rounds=0, rsteps=0, cands=0, lanes_active=0)
    for w in range(ncol):
        mem = cols[w]
        cx, cy = x[mem], y[mem]
        L, own_steps = [], 0
        for l_, i in enumerate(mem):
            l, s, cc = lane_scan([np.inf] * K, x[i], y[i], cx, cy, l_ + 1, l_ - 1)
            L.append(l)
            own_steps = max(own_steps, s)
            st['cands'] += cc
        cost += OWN0 + own_steps * STEP
        st['own'] += own_steps
        # per-lane column sequences
        nxt = [[w - 1, w + 1, 0] for _ in mem]  # lo, hi, side
        while True:
            tasks = []
            for l_, i in enumerate(mem):
                lo, hi, side = nxt[l_]
                found = None
                while lo >= 0 or hi < ncol:
                    c = lo if (side == 0 and lo >= 0) or hi >= ncol else hi
                    if c == lo:
                        gap = np.float32(x[i] - x[(c + 1) * C - 1])
                    else:
                        gap = np.float32(x[c * C] - x[i])
                    if gap < L[l_][K - 1]:
                        found = c
                        if c == lo:
                            lo -= 1
                        else:
                            hi += 1
                        side ^= 1
                        break
                    if c == lo:
                        lo = -1
                    else:
                        hi = ncol
                nxt[l_] = [lo, hi, side]
                if found is not None:
                    tasks.append((l_, found))
            cost += SETUP
            if not tasks:
                break
            st['rounds'] += 1
            st['lanes_active'] += len(tasks)
            ms = 0
            for l_, c in tasks:
                i = mem[l_]
                cm = cols[c]
                start = int(np.sum(yr[cm] < (yr[i] // 32) * 32))
                l, s, cc = lane_scan(L[l_], x[i], y[i], x[cm], y[cm], start, start - 1)
                L[l_] = l
                ms = max(ms, s)
                st['cands'] += cc
            cost += ms * STEP
            st['rsteps'] += ms
        for l_, i in enumerate(mem):
            eps[i] = L[l_][K - 1]
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
    print(f"rounds model {tc / npairs:.0f} warp-ALU per pair vs sweep model {told / npairs:.0f} ({told / tc:.2f}x)")


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
