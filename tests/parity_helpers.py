"""Shared checks of the GPU parity tests (test infrastructure): the region-argmax margin rule and
the oracle enumeration it needs."""
import numpy as np

import oracle


def assert_region_argmax(got_max, got_arg, ref_max, ref_arg, ref_second, tol, value_at):
    """The parity bar for region maxima (BASELINE.json north_star): max within tol; the argmax
    bit-exact whenever the oracle's winning margin (max - best value of any other point pair)
    exceeds tol; otherwise the GPU's argmax must be a valid pair of the region (value_at returns
    its oracle value, None if it is not one of the region's candidates) within tol of the max.
    All-NaN regions: NaN and (-1, -1)."""
    got_max, got_arg = np.asarray(got_max, np.float64), np.asarray(got_arg)
    for r in range(len(ref_max)):
        if np.isnan(ref_max[r]):
            assert np.isnan(got_max[r]) and tuple(got_arg[r]) == (-1, -1), r
            continue
        assert abs(got_max[r] - ref_max[r]) <= tol, (r, got_max[r], ref_max[r])
        ga = (int(got_arg[r][0]), int(got_arg[r][1]))
        if ref_max[r] - ref_second[r] > tol:
            assert ga == tuple(int(v) for v in ref_arg[r]), (r, ga, tuple(ref_arg[r]), ref_max[r] - ref_second[r])
        elif ga != tuple(int(v) for v in ref_arg[r]):
            v = value_at(r, ga)
            assert v is not None and v >= ref_max[r] - tol, (r, ga, v, ref_max[r])


def enumerated_value_at(vals, va, vb):
    """value_at() over an enumerated candidate list (oracle.region_values)."""
    def f(r, ab):
        hit = np.nonzero((va[r] == ab[0]) & (vb[r] == ab[1]))[0]
        if hit.size == 0 or np.isnan(vals[r][hit[0]]):
            return None
        return float(vals[r][hit[0]])
    return f


def oracle_region_reference(fa_vals, fb_vals, dims, measure, k, A, B, samples, seed):
    """(max, argmax, runner-up, value_at) of every region pair from the oracle's enumeration
    (per region pair when exhaustive, so box sizes may differ)."""
    if samples > 0:
        vals, va, vb = oracle.region_values(fa_vals, fb_vals, dims, measure, k, A, B, samples, seed)
        mx, arg, sec = oracle.select_max(vals, va, vb)
        return mx, arg, sec, enumerated_value_at(vals, va, vb)
    if len(A) == 0:
        return np.zeros(0), np.zeros((0, 2), np.int64), np.zeros(0), lambda r, ab: None
    parts = [oracle.region_values(fa_vals, fb_vals, dims, measure, k, [A[r]], [B[r]], 0, seed)
             for r in range(len(A))]
    sel = [oracle.select_max(*p) for p in parts]
    mx = np.array([s_[0][0] for s_ in sel])
    arg = np.array([s_[1][0] for s_ in sel])
    sec = np.array([s_[2][0] for s_ in sel])
    vals = [p[0][0] for p in parts]
    va = [p[1][0] for p in parts]
    vb = [p[2][0] for p in parts]
    return mx, arg, sec, enumerated_value_at(vals, va, vb)


def in_box(p, box, nx, ny):
    x, y, z = p % nx, (p // nx) % ny, p // (nx * ny)
    return box[0] <= x < box[3] and box[1] <= y < box[4] and box[2] <= z < box[5]


