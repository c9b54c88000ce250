"""Cell k-NN cost model with a multi-column own window (development tool, round 2).

Warp = column w (32 x-ranks); its own scan runs over the y-sorted merge of columns
w-h .. w+h (window of 2h+1 columns) from the member's own position; afterwards columns beyond
the window are visited lockstep (lanes that need them), starting at the member's band.
Reports warp steps (1-step lockstep, both directions per step) and column visits per pair.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from sweep_sim import pairs_of  # noqa: E402
from cell_sim import scan, K  # noqa: E402


def pair_stats(x, y, h, C=32):
    n = len(x)
    ncol = (n + C - 1) // C
    yr = np.empty(n, np.int64)
    yr[np.argsort(y, kind="stable")] = np.arange(n)
    cols = [np.arange(c * C, min(n, (c + 1) * C))[np.argsort(yr[c * C:min(n, (c + 1) * C)], kind="stable")]
            for c in range(ncol)]
    own_steps = vis = vsteps = 0
    eps = np.empty(n, np.float32)
    for w in range(ncol):
        mem = cols[w]
        win = np.concatenate([cols[c] for c in range(max(0, w - h), min(ncol, w + h + 1))])
        win = win[np.argsort(yr[win], kind="stable")]
        pos = np.searchsorted(yr[win], yr[mem])
        xi, yi = x[mem], y[mem]
        L = np.full((len(mem), K), np.inf, np.float32)
        L, s = scan(L, yi, xi, x[win], y[win], pos + 1, pos - 1, np.ones(len(mem), bool))
        own_steps += s
        lo, hi = w - h - 1, w + h + 1
        while lo >= 0 or hi < ncol:
            for side in (0, 1):
                c = lo if side == 0 else hi
                if c < 0 or c >= ncol:
                    continue
                gap = np.float32(xi - x[(c + 1) * C - 1]) if side == 0 else np.float32(x[c * C] - xi)
                need = gap < L[:, K - 1]
                if not need.any():
                    if side == 0:
                        lo = -1
                    else:
                        hi = ncol
                    continue
                cm = cols[c]
                start = np.array([np.sum(yr[cm] < (yr[i] // 32) * 32) for i in mem])
                L, s = scan(L, yi, xi, x[cm], y[cm], start, start - 1, need)
                vis += 1
                vsteps += s
                if side == 0:
                    lo -= 1
                else:
                    hi += 1
        eps[mem] = L[:, K - 1]
    return own_steps, vis, vsteps, eps


def main(npairs=4):
    for h in (0, 1, 2):
        tot = np.zeros(3)
        for xa, xb in pairs_of(npairs):
            if xb.std() > xa.std():
                xa, xb = xb, xa
            o = np.argsort(xa, kind="stable")
            x, y = xa[o], xb[o]
            d = np.maximum(np.abs(x[:, None] - x[None, :]), np.abs(y[:, None] - y[None, :]))
            np.fill_diagonal(d, np.inf)
            ref = np.partition(d, K - 1, 1)[:, K - 1]
            a, b, c, e = pair_stats(x, y, h)
            assert np.array_equal(e, ref)
            tot += (a, b, c)
        tot /= npairs
        print(f"window {2 * h + 1} columns: own steps {tot[0]:.0f}, visits {tot[1]:.0f}, visit steps {tot[2]:.0f} per pair")


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
