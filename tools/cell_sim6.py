"""Cell k-NN cost model, variant 'boundary warps' (development tool, round 2).

Warp g owns the 32 members nearest to the boundary between columns g-1 and g (x-ranks
[32g-16, 32g+16)), so its lanes share needs: every lane's nearest neighbour column is the OTHER
column of the pair.  Round 0: every lane scans its own column; then rounds in which every lane
scans its own next needed column (near side first, alternating), lockstep, lanes without a
needed column idle.  Compared with the column warps of ksg_cell_kernel (cell_sim.py)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from sweep_sim import pairs_of  # noqa: E402
from cell_sim2 import lane_scan, K  # noqa: E402


def pair_stats(x, y, C=32):
    n = len(x)
    ncol = (n + C - 1) // C
    yr = np.empty(n, np.int64)
    yr[np.argsort(y, kind="stable")] = np.arange(n)
    cols = [np.arange(c * C, min(n, (c + 1) * C))[np.argsort(yr[c * C:min(n, (c + 1) * C)], kind="stable")]
            for c in range(ncol)]
    posin = np.empty(n, np.int64)
    for c in range(ncol):
        posin[cols[c]] = np.arange(len(cols[c]))
    eps = np.empty(n, np.float32)
    own_steps = rounds = rsteps = 0
    lane_slots = active_slots = 0
    for g in range(ncol + 1):
        mem = np.arange(max(0, 32 * g - 16), min(n, 32 * g + 16))
        if len(mem) == 0:
            continue
        L = [[np.inf] * K for _ in mem]
        ms = 0
        for l_, i in enumerate(mem):
            c = i // C
            p = posin[i]
            l, s, _ = lane_scan(L[l_], x[i], y[i], x[cols[c]], y[cols[c]], p + 1, p - 1)
            L[l_] = l
            ms = max(ms, s)
        own_steps += ms
        # per-lane column sequences: near side first, then alternate
        st = []
        for l_, i in enumerate(mem):
            c = i // C
            near_right = c == g - 1  # a column g-1 member: the boundary is to its right
            st.append({"lo": c - 1, "hi": c + 1, "side": 1 if near_right else 0})
        while True:
            tasks = []
            for l_, i in enumerate(mem):
                s_ = st[l_]
                found = None
                while s_["lo"] >= 0 or s_["hi"] < ncol:
                    side = s_["side"]
                    if side == 0 and s_["lo"] < 0:
                        side = 1
                    if side == 1 and s_["hi"] >= ncol:
                        side = 0
                    cc = s_["lo"] if side == 0 else s_["hi"]
                    gap = np.float32(x[i] - x[(cc + 1) * C - 1]) if side == 0 else np.float32(x[cc * C] - x[i])
                    s_["side"] = side ^ 1
                    if gap < L[l_][K - 1]:
                        found = cc
                        if side == 0:
                            s_["lo"] -= 1
                        else:
                            s_["hi"] += 1
                        break
                    if side == 0:
                        s_["lo"] = -1
                    else:
                        s_["hi"] = ncol
                if found is not None:
                    tasks.append((l_, found))
            if not tasks:
                break
            rounds += 1
            mx = 0
            for l_, cc in tasks:
                i = mem[l_]
                cm = cols[cc]
                start = int(np.sum(yr[cm] < (yr[i] // 32) * 32))
                l, s, _ = lane_scan(L[l_], x[i], y[i], x[cm], y[cm], start, start - 1)
                L[l_] = l
                mx = max(mx, s)
            rsteps += mx
            lane_slots += 32 * mx
        for l_, i in enumerate(mem):
            eps[i] = L[l_][K - 1]
    return own_steps, rounds, rsteps, eps


def main(npairs=4):
    tot = np.zeros(3)
    for xa, xb in pairs_of(npairs):
        if xb.std() > xa.std():
            xa, xb = xb, xa
        o = np.argsort(xa, kind="stable")
        x, y = xa[o], xb[o]
        d = np.maximum(np.abs(x[:, None] - x[None, :]), np.abs(y[:, None] - y[None, :]))
        np.fill_diagonal(d, np.inf)
        ref = np.partition(d, K - 1, 1)[:, K - 1]
        a, b, c, e = pair_stats(x, y)
        assert np.array_equal(e, ref)
        tot += (a, b, c)
    tot /= npairs
    print(f"boundary warps: own steps {tot[0]:.0f}, rounds {tot[1]:.0f}, round steps {tot[2]:.0f} per pair "
          f"(column warps: own 148, visits 136, visit steps 523)")


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
