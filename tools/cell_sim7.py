"""Cell k-NN cost model, variant 'far-visit queue' (development tool, round 2 session 3).

Baseline = ksg_cell_kernel's schedule (cell_sim.py): a warp per 32-x-rank column, lane = member
in y order; own-column lockstep scan, then neighbour columns nearest first, alternating sides,
visited while any lane needs them (x-gap < l[k-1]), each visit a lockstep up/down scan from the
member's y-band cell start.  Variant: after the distance-1 visits (L1, R1) every lane that still
needs a farther column goes to a CTA-wide queue; the queue is processed 32 members per warp in
per-lane rounds (each lane visits ITS nearest still-needed column; a round lasts as long as its
longest scan).  Reports warp scan steps per pair for both and checks eps against brute force.

    python tools/cell_sim7.py [npairs]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from sweep_sim import pairs_of  # noqa: E402

K = 3
C = 32


def ins(L, d):
    L = np.sort(np.concatenate([L, [d]]))[:K]
    return L


def lane_scan(L, xi, yi, cx, cy, up, dn):
    """One lane's up/down scan of a column (y order) from pointers up / dn; returns L, steps."""
    steps = 0
    up_on, dn_on = up < len(cy), dn >= 0
    while up_on or dn_on:
        steps += 1
        if up_on:
            j = up
            d = max(abs(np.float32(xi - cx[j])), abs(np.float32(yi - cy[j])))
            L = ins(L, d)
            stop = np.float32(cy[j] - yi) >= L[K - 1]
            up += 1
            up_on = (not stop) and up < len(cy)
        if dn_on:
            j = dn
            d = max(abs(np.float32(xi - cx[j])), abs(np.float32(yi - cy[j])))
            L = ins(L, d)
            stop = np.float32(yi - cy[j]) >= L[K - 1]
            dn -= 1
            dn_on = (not stop) and dn >= 0
    return L, steps


def pair_stats(x, y):
    n = len(x)
    ncol = (n + C - 1) // C
    yr = np.empty(n, np.int64)
    yr[np.argsort(y, kind="stable")] = np.arange(n)
    cols = [np.arange(c * C, min(n, (c + 1) * C))[np.argsort(yr[c * C:min(n, (c + 1) * C)], kind="stable")]
            for c in range(ncol)]
    start_of = lambda c, i: int(np.sum(yr[cols[c]] < (yr[i] // 32) * 32))  # noqa: E731
    gapL = lambda i, c: np.float32(x[i] - x[(c + 1) * C - 1])  # noqa: E731
    gapR = lambda i, c: np.float32(x[c * C] - x[i])  # noqa: E731
    st = dict(own=0, d1=0, far=0, far_visits=0, far_lanes=0, q_steps=0, q_rounds=0, queued=0, visits=0)
    eps = np.empty(n, np.float32)
    queue = []
    for w in range(ncol):
        mem = cols[w]
        cx, cy = x[mem], y[mem]
        Ls = [np.full(K, np.inf, np.float32) for _ in mem]
        ms = 0
        for l_, i in enumerate(mem):
            Ls[l_], s = lane_scan(Ls[l_], x[i], y[i], cx, cy, l_ + 1, l_ - 1)
            ms = max(ms, s)
        st["own"] += ms
        lo, hi, side, d = w - 1, w + 1, 0, 1
        # baseline visits (alternating, side ends at the first column no lane needs)
        Lb = [L.copy() for L in Ls]
        snap = None
        while lo >= 0 or hi < ncol:
            c = lo if side == 0 else hi
            if 0 <= c < ncol:
                need = [(gapL(i, c) if c < w else gapR(i, c)) < Lb[l_][K - 1] for l_, i in enumerate(mem)]
                if not any(need):
                    if c < w:
                        lo = -1
                    else:
                        hi = ncol
                else:
                    ms = 0
                    for l_, i in enumerate(mem):
                        if need[l_]:
                            s0 = start_of(c, i)
                            cm = cols[c]
                            Lb[l_], s = lane_scan(Lb[l_], x[i], y[i], x[cm], y[cm], s0, s0 - 1)
                            ms = max(ms, s)
                    st["visits"] += 1
                    if abs(c - w) == 1:
                        st["d1"] += ms
                    else:
                        st["far"] += ms
                        st["far_visits"] += 1
                        st["far_lanes"] += sum(need)
                    if c < w:
                        lo -= 1
                    else:
                        hi += 1
            side ^= 1
            if snap is None and (lo < w - 1 or lo < 0) and (hi > w + 1 or hi >= ncol):
                snap = [L.copy() for L in Lb]  # after the distance-1 visits (or their skip)
        for l_, i in enumerate(mem):
            eps[i] = Lb[l_][K - 1]
        if snap is None:
            snap = [L.copy() for L in Lb]
        # variant: lanes still needing a column at distance >= 2 (with their post-d1 lists) queue up
        for l_, i in enumerate(mem):
            L = snap[l_]
            nl = w - 2 >= 0 and gapL(i, w - 2) < L[K - 1]
            nr = w + 2 < ncol and gapR(i, w + 2) < L[K - 1]
            if nl or nr:
                queue.append([i, w, L.copy(), w - 2, w + 2])
    st["queued"] = len(queue)
    # queue processing: 32 members per warp, per-lane rounds
    for g0 in range(0, len(queue), 32):
        grp = queue[g0:g0 + 32]
        while True:
            ms, active = 0, 0
            for q in grp:
                i, w, L, lo, hi = q
                nl = lo >= 0 and gapL(i, lo) < L[K - 1]
                nr = hi < ncol and gapR(i, hi) < L[K - 1]
                if not (nl or nr):
                    continue
                active += 1
                if nl and (not nr or gapL(i, lo) <= gapR(i, hi)):
                    c = lo
                    q[3] -= 1
                else:
                    c = hi
                    q[4] += 1
                s0 = start_of(c, i)
                cm = cols[c]
                q[2], s = lane_scan(L, x[i], y[i], x[cm], y[cm], s0, s0 - 1)
                ms = max(ms, s)
            if active == 0:
                break
            st["q_rounds"] += 1
            st["q_steps"] += ms
        for q in grp:
            assert q[2][K - 1] == eps[q[0]], "variant eps mismatch"
    return st, eps


def main(npairs=4):
    agg = {}
    for xa, xb in pairs_of(npairs):
        if xb.std() > xa.std():
            xa, xb = xb, xa
        o = np.argsort(xa, kind="stable")
        x, y = xa[o], xb[o]
        d = np.maximum(np.abs(x[:, None] - x[None, :]), np.abs(y[:, None] - y[None, :]))
        np.fill_diagonal(d, np.inf)
        ref = np.partition(d, K - 1, 1)[:, K - 1]
        st, eps = pair_stats(x, y)
        assert np.array_equal(eps, ref)
        for k_, v in st.items():
            agg[k_] = agg.get(k_, 0) + v
    print({k_: round(v / npairs, 1) for k_, v in agg.items()})


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
