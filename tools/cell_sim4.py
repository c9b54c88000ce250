"""Fixed-pattern cell k-NN + certificate (development tool, round 2).

Per member i (column c = x-rank // 32, y order inside columns, band b = y-rank // 32):
  own column: the P_own nearest positions above and below in y order (fixed, no stop tests);
  columns c-1 and c+1: positions [s - PD, s + PU) with s = cellstart[col][b] (members of that
  column with y-rank < 32 b), fixed.
Certificate: every direction's last scanned candidate has |dy| >= l[k-1] (or the column ended),
and the x-gap to columns c-2 / c+2 is >= l[k-1].  Members without a certificate go to an exact
fallback.  Reports the failure rate and checks that certified eps equals brute force.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from sweep_sim import pairs_of  # noqa: E402

K = 3


def run(x, y, P_own, PD, PU, C=32):
    n = len(x)
    ncol = (n + C - 1) // C
    yr = np.empty(n, np.int64)
    yr[np.argsort(y, kind="stable")] = np.arange(n)
    cols = [np.arange(c * C, min(n, (c + 1) * C))[np.argsort(yr[c * C:min(n, (c + 1) * C)], kind="stable")]
            for c in range(ncol)]
    pos_in_col = np.empty(n, np.int64)
    for c in range(ncol):
        pos_in_col[cols[c]] = np.arange(len(cols[c]))
    d = np.maximum(np.abs(x[:, None] - x[None, :]), np.abs(y[:, None] - y[None, :]))
    np.fill_diagonal(d, np.inf)
    eps_true = np.partition(d, K - 1, 1)[:, K - 1]
    fail = np.zeros(n, bool)
    reasons = np.zeros(4, np.int64)
    for i in range(n):
        c = i // C
        cands = []
        ok = True
        mem = cols[c]
        p = pos_in_col[i]
        up = mem[p + 1:p + 1 + P_own]
        dn = mem[max(0, p - P_own):p]
        cands += list(up) + list(dn)
        checks = []  # (candidate index or None=column end, sign)
        checks.append((mem[p + P_own] if p + P_own < len(mem) else None, +1, 0))
        checks.append((mem[p - P_own] if p - P_own >= 0 else None, -1, 0))
        for cc in (c - 1, c + 1):
            if cc < 0 or cc >= ncol:
                continue
            m2 = cols[cc]
            s = int(np.sum(yr[m2] < (yr[i] // 32) * 32))
            lo, hi = max(0, s - PD), min(len(m2), s + PU)
            cands += list(m2[lo:hi])
            checks.append((m2[hi - 1] if hi < len(m2) else None, +1, 1))
            checks.append((m2[lo] if lo > 0 else None, -1, 1))
        l2 = np.sort(d[i, cands])[K - 1] if len(cands) >= K else np.inf
        for j, sg, r in checks:
            if j is None:
                continue
            dy = np.float32(y[j] - y[i]) if sg > 0 else np.float32(y[i] - y[j])
            if not dy >= l2:
                ok = False
                reasons[r] += 1
        for cc, side in ((c - 2, 0), (c + 2, 1)):
            if 0 <= cc < ncol:
                gap = np.float32(x[i] - x[(cc + 1) * C - 1]) if side == 0 else np.float32(x[cc * C] - x[i])
                if not gap >= l2:
                    ok = False
                    reasons[2] += 1
        if ok:
            assert l2 == eps_true[i], (i, l2, eps_true[i])
        fail[i] = not ok
    return fail.mean(), reasons


def main(npairs=6):
    pairs = pairs_of(npairs)
    for P_own, PD, PU in ((2, 2, 3), (3, 2, 3), (3, 3, 4), (4, 3, 4), (4, 4, 5), (5, 4, 6)):
        fr, rs = [], np.zeros(4, np.int64)
        for xa, xb in pairs:
            if xb.std() > xa.std():
                xa, xb = xb, xa
            o = np.argsort(xa, kind="stable")
            f, r = run(xa[o], xb[o], P_own, PD, PU)
            fr.append(f)
            rs += r
        cands = 2 * P_own + 2 * (PD + PU)
        print(f"P_own={P_own} PD={PD} PU={PU} cands={cands}: fail {np.mean(fr):.3f} reasons(own,nbr,gap2)={rs[:3] / npairs}")


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 6)
