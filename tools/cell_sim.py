"""SIMT cost model of a column-cell k-NN for KSG (development tool, round 2).

Layout per staged pair (x = the wider marginal): members in x order are cut into columns of C
consecutive x-ranks; inside a column the members are kept in y order.  A warp owns one column,
lane l = the column's l-th member in y order.  Per member:
  own column   -- scan up (l+1, l+2, ...) and down (l-1, ...) in y order, one candidate per
                  direction per step; a direction stops once fl(y_j - y_i) >= l_i[k-1] (all
                  further ones are farther in y), or at the column end;
  neighbour columns, nearest first, alternating sides -- the column is needed iff
                  fl(x-gap to its nearest x) < l_i[k-1] for some lane; needing lanes binary-search
                  y_i in the column's y order and scan up/down from there with the same stop rule.
A warp step costs STEP warp-ALU instructions for all lanes (max over the lanes' step counts),
a column visit SEARCH + COLTEST.  Every schedule is checked to reproduce brute-force eps.

    python tools/cell_sim.py [npairs] [C]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from sweep_sim import pairs_of, warp_cost  # noqa: E402

K = 3
STEP, SEARCH, COLTEST = 14.0, 10.0, 3.0


def insert(L, d):
    return np.sort(np.concatenate([L, d[:, None]], 1), 1)[:, :K]


def scan(L, yi, xi, cx, cy, start_up, start_dn, active):
    """Lockstep up/down scan of one column for the active lanes; returns (L, warp steps)."""
    nl = len(yi)
    u, dn = start_up.copy(), start_dn.copy()
    up_on = active & (u < len(cy))
    dn_on = active & (dn >= 0)
    steps = 0
    while up_on.any() or dn_on.any():
        steps += 1
        for on, ptr, sgn in ((up_on, u, 1), (dn_on, dn, -1)):
            idx = np.where(on)[0]
            if len(idx) == 0:
                continue
            j = ptr[idx]
            dy = np.float32(cy[j] - yi[idx]) if sgn > 0 else np.float32(yi[idx] - cy[j])
            d = np.maximum(np.abs(np.float32(xi[idx] - cx[j])), np.abs(np.float32(yi[idx] - cy[j])))
            Lsub = insert(L[idx], d)
            L[idx] = Lsub
            stop = dy >= L[idx, K - 1]
            ptr[idx] = j + sgn
            on[idx] = ~stop & ((ptr[idx] < len(cy)) if sgn > 0 else (ptr[idx] >= 0))
    return L, steps


def pair_cost(x, y, C):
    n = len(x)
    ncol = (n + C - 1) // C
    cols = []
    for c in range(ncol):
        t = np.arange(c * C, min(n, (c + 1) * C))
        o = t[np.argsort(y[t], kind="stable")]
        cols.append(o)
    cost = 0.0
    eps = np.empty(n, np.float32)
    steps_tot = 0
    cand = 0
    for w in range(ncol):
        mem = cols[w]
        xi, yi = x[mem], y[mem]
        nl = len(mem)
        L = np.full((nl, K), np.inf, np.float32)
        cx, cy = x[mem], y[mem]
        lanes = np.arange(nl)
        L, s = scan(L, yi, xi, cx, cy, lanes + 1, lanes - 1, np.ones(nl, bool))
        cost += s * STEP
        steps_tot += s
        lo, hi = w - 1, w + 1
        side = 0
        while lo >= 0 or hi < ncol:
            for c in ((lo,) if side == 0 else (hi,)):
                if c < 0 or c >= ncol:
                    continue
                cm = cols[c]
                cost += COLTEST
                if c < w:
                    gap = np.float32(xi - x[(c + 1) * C - 1])
                else:
                    gap = np.float32(x[c * C] - xi)
                need = gap < L[:, K - 1]
                if not need.any():
                    if c < w:
                        lo = -1
                    else:
                        hi = ncol
                    continue
                ccx, ccy = x[cm], y[cm]
                pos = np.searchsorted(ccy, yi, side="left")
                cost += SEARCH
                L, s = scan(L, yi, xi, ccx, ccy, pos, pos - 1, need)
                cost += s * STEP
                steps_tot += s
                cand += 2 * s
                if c < w:
                    lo -= 1
                else:
                    hi += 1
            side ^= 1
        eps[mem] = L[:, K - 1]
    return cost, eps, steps_tot


def main(npairs=12, C=32):
    tc, told = 0.0, 0.0
    for xa, xb in pairs_of(npairs):
        if xb.std() > xa.std():
            xa, xb = xb, xa
        o = np.argsort(xa, kind="stable")
        x, y = xa[o], xb[o]
        n = len(x)
        d = np.maximum(np.abs(x[:, None] - x[None, :]), np.abs(y[:, None] - y[None, :]))
        np.fill_diagonal(d, np.inf)
        eps = np.partition(d, K - 1, 1)[:, K - 1]
        c, e, st = pair_cost(x, y, C)
        assert np.array_equal(e, eps)
        old = 0.0
        for b0 in range(0, n, 32):
            cw, _, _ = warp_cost(x, y, b0, 32, 1, 32, False)
            old += cw
        tc += c
        told += old
        print(f"pair: cell {c:8.0f}  sweep {old:8.0f}  ratio {old / c:.2f}", flush=True)
    print(f"C={C}: cell model {tc / npairs:.0f} warp-ALU per pair vs sweep model {told / npairs:.0f} "
          f"({told / tc:.2f}x)")


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 12, int(sys.argv[2]) if len(sys.argv) > 2 else 32)
