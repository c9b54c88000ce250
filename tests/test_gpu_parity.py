"""GPU parity: libcorr.so (through the C ABI) vs the CPU oracle on identical generator bytes.

Bars (BASELINE.json north_star): eps and marginal counts bit-exact; KSG MI within 1e-4;
Pearson within 1e-5; region argmax bit-exact whenever the winning margin exceeds the
tolerance (otherwise the GPU's argmax must be a pair whose oracle value is within
tolerance of the max).
"""
import math

import numpy as np
import pytest
import torch

import oracle
from paper_2309_03308_b200 import binding as cb
from paper_2309_03308_b200 import synth
from parity_helpers import assert_region_argmax, in_box, oracle_region_reference

pytestmark = pytest.mark.gpu

KSG_TOL = 1e-4
PEARSON_TOL = 1e-5


def _field(spec, device="cuda"):
    vals = synth.generate(spec, device=device)
    f = cb.corr_field_create(vals, spec.nx, spec.ny, spec.nz, spec.members)
    return vals, f


def _cpu(t):
    return t.detach().cpu().numpy()


def test_generator_bytes_identical_on_cpu_and_cuda():
    spec = synth.spec_of(synth.C1)
    assert torch.equal(synth.generate(spec, "cuda").cpu(), synth.generate(spec, "cpu"))
    spec = synth.spec_of(synth.C3)
    pts = torch.tensor([0, 17, 123456, spec.points - 1])
    assert torch.equal(synth.rows(spec, pts.cuda()).cpu(), synth.rows(spec, pts))


def _all_pairs(P):
    a, b = np.triu_indices(P, 1)
    return a.astype(np.int64), b.astype(np.int64)


@pytest.mark.parametrize("measure", [oracle.KSG, oracle.KSG | oracle.F_KSG_PLUS1, oracle.PEARSON])
def test_c1_all_point_pairs(measure):
    spec = synth.spec_of(synth.C1)
    vals, f = _field(spec)
    a, b = _all_pairs(spec.points)  # 32 640 pairs
    ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    got = _cpu(cb.corr_eval_pairs(f, None, measure, 3, ta, tb))
    cb.corr_check(f)
    ref = oracle.eval_pairs(vals.cpu(), None, measure, 3, a, b)
    tol = PEARSON_TOL if measure == oracle.PEARSON else KSG_TOL
    assert np.array_equal(np.isnan(got), np.isnan(ref))
    ok = ~np.isnan(ref)
    assert np.max(np.abs(got[ok] - ref[ok])) <= tol


def _check_knn(f, vals, k, a, b, fb=None, vals_b=None):
    ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    eps, nx, ny = cb.corr_ksg_debug(f, fb, k, ta, tb)
    cb.corr_check(f)
    reps, rnx, rny = oracle.knn_pairs(vals.cpu(), None if vals_b is None else vals_b.cpu(), k, a, b)
    assert np.array_equal(_cpu(eps), reps)
    assert np.array_equal(_cpu(nx), rnx)
    assert np.array_equal(_cpu(ny), rny)


def test_c1_eps_counts_bit_exact():
    spec = synth.spec_of(synth.C1)
    vals, f = _field(spec)
    a, b = _all_pairs(spec.points)
    _check_knn(f, vals, 3, a[::7], b[::7])


@pytest.mark.parametrize("n,k,dims", [(100, 3, (16, 16, 4)), (1000, 3, (8, 8, 4)), (37, 1, (8, 8, 2)),
                                      (130, 5, (8, 8, 2)), (257, 8, (8, 4, 2)), (1001, 4, (4, 4, 2)),
                                      (4, 3, (8, 8, 1)), (129, 2, (8, 4, 2)), (1000, 30, (4, 4, 2)),
                                      (200, 12, (8, 4, 2)), (300, 17, (8, 4, 2)), (1000, 0, (4, 4, 2)),
                                      (64, 32, (8, 4, 2)), (500, 31, (4, 4, 2)), (700, 25, (4, 4, 2)),
                                      (129, 30, (4, 4, 2))])
def test_eps_counts_mi_bit_exact_ragged(n, k, dims):
    """k = 0 selects the paper's ceil(3n/100); k > 8 uses the long-list kernels."""
    spec = synth.field_spec(*dims, n, seed=100 + n)
    vals, f = _field(spec)
    a, b = synth.random_pairs(spec.points, 300 if n <= 300 else 60, seed=n)
    a, b = a.numpy(), b.numpy()
    kk = k if k else min(max(1, -(-3 * n // 100)), n - 1)
    _check_knn(f, vals, kk, a, b)
    if k == 0:
        e0, _, _ = cb.corr_ksg_debug(f, None, 0, torch.from_numpy(a[:4]).cuda(), torch.from_numpy(b[:4]).cuda())
        e1, _, _ = cb.corr_ksg_debug(f, None, kk, torch.from_numpy(a[:4]).cuda(), torch.from_numpy(b[:4]).cuda())
        assert torch.equal(e0, e1)
    k = kk
    got = _cpu(cb.corr_eval_pairs(f, None, cb.CORR_KSG, k, torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()))
    ref = oracle.eval_pairs(vals.cpu(), None, oracle.KSG, k, a, b)
    assert np.array_equal(np.isnan(got), np.isnan(ref))
    ok = ~np.isnan(ref)
    assert np.max(np.abs(got[ok] - ref[ok]), initial=0) <= KSG_TOL
    got = _cpu(cb.corr_eval_pairs(f, None, cb.CORR_PEARSON, 0, torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()))
    ref = oracle.eval_pairs(vals.cpu(), None, oracle.PEARSON, 0, a, b)
    assert np.max(np.abs(got - ref)) <= PEARSON_TOL


def test_ties_zero_inflated_and_constant_series():
    """hail/precip-like fields: 60% exact zeros (eps = 0 -> counts 0 -> psi(0) -> NaN)."""
    n, P = 100, 64
    g = torch.Generator().manual_seed(5)
    vals = torch.rand((n, P), generator=g)
    vals[torch.rand((n, P), generator=g) < 0.6] = 0.0
    vals[:, 3] = 2.5  # constant series
    vals = vals.contiguous()
    f = cb.corr_field_create(vals.cuda(), 8, 8, 1, n)
    a, b = synth.random_pairs(P, 400, seed=9)
    a, b = a.numpy(), b.numpy()
    a[:5] = 3
    _check_knn(f, vals, 3, a[5:], b[5:])
    for measure in (oracle.KSG, oracle.KSG | oracle.F_KSG_PLUS1, oracle.PEARSON):
        got = _cpu(cb.corr_eval_pairs(f, None, measure, 3, torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()))
        ref = oracle.eval_pairs(vals, None, measure, 3, a, b)
        assert np.array_equal(np.isnan(got), np.isnan(ref)), measure
        ok = ~np.isnan(ref)
        tol = PEARSON_TOL if measure == oracle.PEARSON else KSG_TOL
        assert np.max(np.abs(got[ok] - ref[ok]), initial=0) <= tol
        assert np.isnan(got[:5]).all()


def test_out_of_range_index_flagged():
    spec = synth.spec_of(synth.C1)
    vals, f = _field(spec)
    a = torch.tensor([0, 1, 9999], dtype=torch.int64, device="cuda")
    b = torch.tensor([5, 6, 7], dtype=torch.int64, device="cuda")
    out = cb.corr_eval_pairs(f, None, cb.CORR_KSG, 3, a, b)
    with pytest.raises(cb.CorrError) as e:
        cb.corr_check(f)
    assert e.value.code == cb.CORR_E_RANGE
    assert math.isnan(out[2].item()) and not math.isnan(out[0].item())
    cb.corr_check(f)  # flag cleared


def test_invalid_arguments():
    spec = synth.spec_of(synth.C1)
    vals, f = _field(spec)
    a = torch.zeros(2, dtype=torch.int64, device="cuda")
    with pytest.raises(cb.CorrError):
        cb.corr_eval_pairs(f, None, cb.CORR_KSG, 10, a, a)  # k > n-1
    with pytest.raises(cb.CorrError):
        cb.corr_region_max(f, None, cb.CORR_KSG, 3, [(0, 0, 0, 0, 1, 1)], [(0, 0, 0, 1, 1, 1)], 10, 1)
    with pytest.raises(cb.CorrError):
        cb.corr_region_max(f, None, cb.CORR_KSG, 3, [(0, 0, 0, 9, 1, 1)], [(0, 0, 0, 1, 1, 1)], 10, 1)
    bad = vals.clone()
    bad[3, 7] = float("nan")
    with pytest.raises(cb.CorrError):
        cb.corr_field_create(bad, 8, 8, 4, 10)


def _region_compare(got_max, got_arg, fa_vals, fb_vals, dims, measure, k, A, B, samples, seed, tol):
    mx, arg, sec, value_at = oracle_region_reference(fa_vals, fb_vals, dims, measure, k, A, B, samples, seed)
    # the oracle's C region_max agrees with the enumeration (same max / argmax)
    rmx, rarg = oracle.region_max(fa_vals, fb_vals, dims, measure, k, A, B, samples, seed)
    assert np.array_equal(rmx, mx, equal_nan=True) and np.array_equal(rarg, arg)
    assert_region_argmax(_cpu(got_max), _cpu(got_arg), mx, arg, sec, tol, value_at)


@pytest.mark.parametrize("measure", [oracle.KSG, oracle.PEARSON, oracle.PEARSON | oracle.F_ABS,
                                     oracle.KSG | oracle.F_KSG_PLUS1])
@pytest.mark.parametrize("samples", [0, 37])
def test_c1_region_max(measure, samples):
    spec = synth.spec_of(synth.C1)
    vals, f = _field(spec)
    A, B = synth.context_pairs(synth.bricks_of(synth.C1))
    got_max, got_arg = cb.corr_region_max(f, None, measure, 3, A, B, samples, 1234)
    tol = PEARSON_TOL if (measure & 0xFF) == oracle.PEARSON else KSG_TOL
    _region_compare(got_max, got_arg, vals.cpu(), None, (8, 8, 4), measure, 3, A, B, samples, 1234, tol)


def test_c1_two_field_matrix_region_max():
    """Inter-variable matrix: ordered region pairs across two fields."""
    cfg = synth.C1
    sa, sb = synth.spec_of(cfg, 1), synth.spec_of(cfg, 2)
    va, fa = _field(sa)
    vb, fb = _field(sb)
    A, B = synth.matrix_pairs(synth.bricks_of(cfg))
    for measure, samples in ((oracle.PEARSON, 0), (oracle.KSG, 0), (oracle.KSG, 25)):
        got_max, got_arg = cb.corr_region_max(fa, fb, measure, 3, A, B, samples, 77)
        tol = PEARSON_TOL if measure == oracle.PEARSON else KSG_TOL
        _region_compare(got_max, got_arg, va.cpu(), vb.cpu(), (8, 8, 4), measure, 3, A, B, samples, 77, tol)


def _block_compare(f, fb, vals_a, vals_b, dims, A, B, absval=False):
    """Exhaustive Pearson region max vs the oracle's block max (fp64 library matmul), with the
    argmax-margin rule (the oracle's runner-up over every other point pair)."""
    measure = cb.CORR_PEARSON | (cb.CORR_F_ABS if absval else 0)
    got_max, got_arg = cb.corr_region_max(f, fb, measure, 0, A, B, 0, 0)
    cb.corr_check(f)
    got_max, got_arg = _cpu(got_max), _cpu(got_arg)
    ref = [oracle.pearson_block_max(vals_a, vals_b, dims, A[r], B[r], absval=absval, runner_up=True)
           for r in range(len(A))]

    def value_at(r, ab):
        if not (in_box(ab[0], A[r], dims[0], dims[1]) and in_box(ab[1], B[r], dims[0], dims[1])):
            return None
        if fb is None and ab[0] == ab[1]:
            return None
        w = oracle.eval_pairs(vals_a, vals_b, oracle.PEARSON, 0, [ab[0]], [ab[1]])[0]
        w = float(np.float32(abs(w) if absval else w))
        return None if np.isnan(w) else w

    assert_region_argmax(got_max, got_arg, np.array([v[0] for v in ref]), np.array([v[1] for v in ref]),
                         np.array([v[2] for v in ref]), PEARSON_TOL, value_at)


def test_pearson_block_c2_focus_full():
    """C2: all 20 480^2 = 4.2e8 point pairs of the two focus bricks, n = 100, tcgen05 path."""
    spec = synth.spec_of(synth.C2)
    vals, f = _field(spec)
    host = vals.cpu().numpy()
    _block_compare(f, None, host, None, (spec.nx, spec.ny, spec.nz), [synth.C2_REGION_A], [synth.C2_REGION_B])
    got_max, _ = cb.corr_region_max(f, None, cb.CORR_PEARSON, 0, [synth.C2_REGION_A], [synth.C2_REGION_B], 0, 0)
    assert abs(float(got_max[0]) - 1.0) <= 1e-6  # cluster centres share one signal


def test_pearson_block_context_boundary_and_overlap():
    spec = synth.spec_of(synth.C3)
    vals, f = _field(spec)
    host = vals.cpu().numpy()
    bricks = synth.bricks_of(synth.C3)
    A = [bricks[7], bricks[0], bricks[15], bricks[40], (100, 100, 3, 164, 110, 9)]
    B = [bricks[80], bricks[87], bricks[16], bricks[40], (120, 96, 0, 150, 140, 20)]
    _block_compare(f, None, host, None, (spec.nx, spec.ny, spec.nz), A, B)
    _block_compare(f, None, host, None, (spec.nx, spec.ny, spec.nz), A[:3], B[:3], absval=True)


def test_pearson_block_odd_tile_counts_and_z_split():
    """Boxes whose A side has an ODD number of 128-point tiles (the multicast screen pairs A tiles
    per cluster and duplicates the last one) and whose B tiles are split along z between the two
    CTAs of a cluster (small x/y extents), plus an overlapping (self-pair masked) box pair."""
    spec = synth.spec_of(synth.C3)
    vals, f = _field(spec)
    host = vals.cpu().numpy()
    A = [(0, 0, 0, 16, 8, 3), (40, 50, 2, 56, 58, 11), (0, 0, 0, 16, 8, 3)]
    B = [(100, 100, 0, 108, 108, 20), (10, 20, 5, 18, 28, 9), (4, 2, 0, 12, 10, 4)]
    _block_compare(f, None, host, None, (spec.nx, spec.ny, spec.nz), A, B)
    _block_compare(f, None, host, None, (spec.nx, spec.ny, spec.nz), A, B, absval=True)


def test_pearson_block_n1000_and_two_fields():
    cfg = synth.C5
    sa, sb = synth.spec_of(cfg, 1), synth.spec_of(cfg, 2)
    va, fa = _field(sa)
    vb, fb = _field(sb)
    ha, hb = va.cpu().numpy(), vb.cpu().numpy()
    del va, vb
    A = [(8, 8, 5, 40, 16, 10), (160, 232, 8, 192, 248, 12)]
    B = [(170, 230, 8, 202, 238, 13), (0, 0, 0, 16, 16, 5)]
    _block_compare(fa, fb, ha, hb, (sa.nx, sa.ny, sa.nz), A, B)
    _block_compare(fa, None, ha, None, (sa.nx, sa.ny, sa.nz), A, B)


@pytest.mark.parametrize("n,k,npairs", [(2500, 3, 12), (2500, 32, 8), (4096, 5, 3), (20, 19, 60), (40, 32, 60)])
def test_large_n_and_extreme_k(n, k, npairs):
    """Member counts beyond one CTA pass (n up to the 4096 limit) and k = n-1 / k = 32 (the largest
    register list)."""
    spec = synth.field_spec(4, 4, 2, n, seed=n + k)
    vals, f = _field(spec)
    a, b = synth.random_pairs(spec.points, npairs, seed=k)
    a, b = a.numpy(), b.numpy()
    _check_knn(f, vals, k, a, b)
    got = _cpu(cb.corr_eval_pairs(f, None, cb.CORR_KSG, k, torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()))
    ref = oracle.eval_pairs(vals.cpu(), None, oracle.KSG, k, a, b)
    assert np.max(np.abs(got - ref)) <= KSG_TOL


def test_degenerate_boxes_and_limits():
    spec = synth.spec_of(synth.C1)
    vals, f = _field(spec)
    one = (3, 3, 1, 4, 4, 2)
    m, arg = cb.corr_region_max(f, None, cb.CORR_PEARSON, 0, [one], [one], 0, 0)  # only the self pair
    assert math.isnan(float(m[0])) and arg[0].tolist() == [-1, -1]
    m, arg = cb.corr_region_max(f, None, cb.CORR_KSG, 3, [one], [one], 5, 0)
    assert math.isnan(float(m[0])) and arg[0].tolist() == [-1, -1]
    two = (0, 0, 0, 1, 1, 1)
    for measure in (cb.CORR_KSG, cb.CORR_PEARSON):
        m, arg = cb.corr_region_max(f, None, measure, 3, [two], [one], 1, 9)  # a single sample
        ref, rarg = oracle.region_max(vals.cpu(), None, (8, 8, 4), measure, 3, [two], [one], 1, 9)
        assert abs(float(m[0]) - ref[0]) <= KSG_TOL and arg[0].tolist() == list(rarg[0])
    z, o = torch.zeros(1, dtype=torch.int64, device="cuda"), torch.ones(1, dtype=torch.int64, device="cuda")
    v9 = cb.corr_eval_pairs(f, None, cb.CORR_KSG, 9, z, o)  # k = n - 1 is the largest valid k
    assert abs(float(v9[0]) - oracle.eval_pairs(vals.cpu(), None, oracle.KSG, 9, [0], [1])[0]) <= KSG_TOL
    with pytest.raises(cb.CorrError):
        cb.corr_eval_pairs(f, None, cb.CORR_KSG, 10, z, o)
    big = synth.field_spec(350, 200, 1, 4, seed=1)  # 70 000 points
    bv, bf = _field(big)
    full = (0, 0, 0, 350, 200, 1)
    with pytest.raises(cb.CorrError) as e:
        cb.corr_region_max(bf, None, cb.CORR_PEARSON, 0, [full], [full], 0, 0)  # |A||B| >= 2^32
    assert e.value.code == cb.CORR_E_INVAL


def test_field_update_equals_fresh_create():
    """corr_field_update (next ensemble, same shape, no reallocation) gives bit-identical results to
    a field created from the same values; host and device inputs; non-finite input rejected."""
    s1 = synth.field_spec(24, 16, 8, 100, seed=5)
    s2 = synth.field_spec(24, 16, 8, 100, seed=6)
    v1, v2 = synth.generate(s1, device="cuda"), synth.generate(s2, device="cuda")
    f = cb.corr_field_create(v1, s1.nx, s1.ny, s1.nz, s1.members)
    g = cb.corr_field_create(v2, s2.nx, s2.ny, s2.nz, s2.members)
    a, b = synth.random_pairs(s1.points, 300, seed=4)
    a, b = a.cuda(), b.cuda()
    for src in (v2, v2.cpu().pin_memory(), v2.cpu()):
        cb.corr_field_update(f, src)
        for measure in (cb.CORR_KSG, cb.CORR_PEARSON):
            assert torch.equal(cb.corr_eval_pairs(f, None, measure, 3, a, b),
                               cb.corr_eval_pairs(g, None, measure, 3, a, b))
        bricks = synth.partition(s1.nx, s1.ny, s1.nz, 8, 8, 4)
        A, B = synth.context_pairs(bricks)
        m1, a1 = cb.corr_region_max(f, None, cb.CORR_PEARSON, 0, A, B, 0, 0)
        m2, a2 = cb.corr_region_max(g, None, cb.CORR_PEARSON, 0, A, B, 0, 0)
        assert torch.equal(m1, m2) and torch.equal(a1, a2)
    bad = v1.clone()
    bad[1, 2] = float("inf")
    for src in (bad, bad.cpu().pin_memory()):
        cb.corr_field_update(f, src)  # asynchronous: the device flag is reported by corr_check
        with pytest.raises(cb.CorrError) as e:
            cb.corr_check(f)
        assert e.value.code == cb.CORR_E_INVAL
    cb.corr_field_update(f, v1)
    cb.corr_check(f)


def test_invariances_on_gpu_path():
    """the oracle's bit-exact invariances re-run on the GPU path -- swap of
    the two series (Eq. 1 symmetry), a common power-of-two scale, reflection of one field."""
    spec = synth.field_spec(40, 30, 10, 1000, seed=77)
    vals = synth.generate(spec, device="cuda")
    f = cb.corr_field_create(vals, spec.nx, spec.ny, spec.nz, spec.members)
    f4 = cb.corr_field_create((vals * 4.0).contiguous(), spec.nx, spec.ny, spec.nz, spec.members)
    fneg = cb.corr_field_create((-vals).contiguous(), spec.nx, spec.ny, spec.nz, spec.members)
    a, b = synth.random_pairs(spec.points, 500, seed=3)
    a, b = a.cuda(), b.cuda()
    for measure in (cb.CORR_KSG, cb.CORR_KSG | cb.CORR_F_KSG_PLUS1, cb.CORR_PEARSON):
        base = cb.corr_eval_pairs(f, None, measure, 3, a, b)
        assert torch.equal(base, cb.corr_eval_pairs(f, None, measure, 3, b, a))       # swap
        assert torch.equal(base, cb.corr_eval_pairs(f4, None, measure, 3, a, b))      # 2^2 scale
        refl = cb.corr_eval_pairs(fneg, f, measure, 3, a, b)                          # x -> -x
        assert torch.equal(base, -refl if measure == cb.CORR_PEARSON else refl)
    for g in (f, f4, fneg):
        g.close()


def test_dense_and_sweep_identical():
    """The column-cell k-NN (default), the round-1 sweep (CORR_F_KSG_SWEEP), the counting build
    (CORR_F_KSG_COUNT) and CORR_F_KSG_DENSE give bit-identical results."""
    spec = synth.spec_of(synth.C4)
    vals, f = _field(spec)
    del vals
    A, B = synth.context_pairs(synth.bricks_of(synth.C4))
    A, B = A[::40], B[::40]
    for k in (3, 30):
        m1, a1 = cb.corr_region_max(f, None, cb.CORR_KSG, k, A, B, 8, 5)
        m2, a2 = cb.corr_region_max(f, None, cb.CORR_KSG | cb.CORR_F_KSG_DENSE, k, A, B, 8, 5)
        m3, a3 = cb.corr_region_max(f, None, cb.CORR_KSG | cb.CORR_F_KSG_SWEEP, k, A, B, 8, 5)
        m4, a4 = cb.corr_region_max(f, None, cb.CORR_KSG | cb.CORR_F_KSG_COUNT, k, A, B, 8, 5)
        assert torch.equal(m1, m2) and torch.equal(a1, a2)
        assert torch.equal(m1, m3) and torch.equal(a1, a3)  # column-cell k-NN == round-1 sweep
        assert torch.equal(m1, m4) and torch.equal(a1, a4)  # the counting build: same results
    f.close()


def test_focus_sub_brick_matrix():
    """NEXT #3: the (M/2)^2 focus matrix of sub-brick pair maxima in one call; the
    sub-bricks partition the parent bricks, so the matrix max is the parent pair max (same pair)."""
    spec = synth.spec_of(synth.C2)
    vals, f = _field(spec)
    host = vals.cpu().numpy()
    kids_a, kids_b = synth.refine(synth.C2_REGION_A, 44), synth.refine(synth.C2_REGION_B, 44)
    assert len(kids_a) == 8 and sum(synth.box_size(b) for b in kids_a) == synth.box_size(synth.C2_REGION_A)
    A = [a for a in kids_a for _ in kids_b]
    B = [b for _ in kids_a for b in kids_b]
    sm, sa = cb.corr_region_max(f, None, cb.CORR_PEARSON, 0, A, B, 0, 0)
    pm, pa = cb.corr_region_max(f, None, cb.CORR_PEARSON, 0, [synth.C2_REGION_A], [synth.C2_REGION_B], 0, 0)
    assert float(sm.max()) == float(pm[0])
    for r in (0, 9, 63):
        v, ab = oracle.pearson_block_max(host, None, (spec.nx, spec.ny, spec.nz), A[r], B[r])
        assert abs(float(sm[r]) - v) <= PEARSON_TOL


@pytest.mark.parametrize("fac", [(2, 2, 2), (4, 4, 4), (3, 2, 5)])
def test_mean_tree_aggregate(fac):
    """NEXT #4: block means on the GPU equal the oracle's, and region maxima
    computed on the aggregate match the oracle run on the oracle's aggregate."""
    spec = synth.field_spec(32, 24, 10, 100, seed=41)
    vals, f = _field(spec)
    g = cb.corr_field_aggregate(f, *fac)
    dims = (g.nx, g.ny, g.nz)
    ref = oracle.aggregate_mean(vals.cpu(), (spec.nx, spec.ny, spec.nz), *fac)
    # the aggregate's rows, read back through Pearson of a series with itself is not a value
    # check -- compare the KSG eps (bit-exact) and Pearson (1e-5) of random pairs instead
    a, b = synth.random_pairs(g.points, 200, seed=5)
    _check_knn(g, torch.from_numpy(ref), 3, a.numpy(), b.numpy())
    got = _cpu(cb.corr_eval_pairs(g, None, cb.CORR_PEARSON, 0, a.cuda(), b.cuda()))
    assert np.max(np.abs(got - oracle.eval_pairs(ref, None, oracle.PEARSON, 0, a, b))) <= PEARSON_TOL
    boxes = synth.partition(*dims, 8, 8, 5)
    A, B = synth.context_pairs(boxes)
    for measure, S in ((cb.CORR_KSG, 50), (cb.CORR_PEARSON, 0)):
        gm, ga = cb.corr_region_max(g, None, measure, 3, A, B, S, 3)
        tol = PEARSON_TOL if measure == cb.CORR_PEARSON else KSG_TOL
        _region_compare(gm, ga, ref, None, dims, measure, 3, A, B, S, 3, tol)


def test_shards_bit_identical_to_unsharded():
    """1-GPU emulation of the R-GPU split: shards run one after the
    other and concatenated equal the unsharded call bit for bit (sampler keyed by boxes)."""
    from paper_2309_03308_b200 import dist as cdist
    spec = synth.spec_of(synth.C3)
    vals, f = _field(spec)
    del vals
    A, B = synth.context_pairs(synth.bricks_of(synth.C3))
    A, B = A[:400], B[:400]
    for measure, S in ((cb.CORR_KSG, 64), (cb.CORR_PEARSON, 64), (cb.CORR_PEARSON, 0)):
        if S == 0:
            A2, B2 = A[:12], B[:12]
        else:
            A2, B2 = A, B
        full_m, full_a = cb.corr_region_max(f, None, measure, 3, A2, B2, S, 99)
        for world in (2, 3, 8):
            ms, as_ = [], []
            for lo, hi in cdist.shard_bounds([1] * len(A2), world):
                m, a = cb.corr_region_max(f, None, measure, 3, A2[lo:hi], B2[lo:hi], S, 99)
                ms.append(m)
                as_.append(a)
            assert torch.equal(torch.cat(ms), full_m) and torch.equal(torch.cat(as_), full_a)


@pytest.mark.parametrize("n", [33, 34, 63, 65, 96, 97, 127, 128])
def test_warp_kernel_partial_chunks(n):
    """n < 128 runs one warp per pair (ksg_warp_kernel) and scans only the existing members of the
    partial last chunk / own block (n = 33: one member, 63: 31); n = 128 is the first CTA-kernel
    size.  eps / counts bit-exact, MI within tolerance, sweep == dense bit for bit."""
    spec = synth.field_spec(8, 4, 2, n, seed=7 * n)
    vals, f = _field(spec)
    a, b = synth.random_pairs(spec.points, 200, seed=n)
    a, b = a.numpy(), b.numpy()
    ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    for k in (1, 3, 8):
        _check_knn(f, vals, k, a, b)
        got = _cpu(cb.corr_eval_pairs(f, None, cb.CORR_KSG, k, ta, tb))
        dense = _cpu(cb.corr_eval_pairs(f, None, cb.CORR_KSG | cb.CORR_F_KSG_DENSE, k, ta, tb))
        ref = oracle.eval_pairs(vals.cpu(), None, oracle.KSG, k, a, b)
        assert np.array_equal(got, dense, equal_nan=True)
        assert np.array_equal(np.isnan(got), np.isnan(ref))
        ok = ~np.isnan(ref)
        assert np.max(np.abs(got[ok] - ref[ok]), initial=0) <= KSG_TOL
    f.close()


@pytest.mark.parametrize("k", [30, 31])
def test_batched_large_k_two_fields_and_dense(k):
    """The batched 32-list path (24 < k <= 31) on TWO fields (x from one variable, y from the
    other; the sort marginal swaps per pair) and with CORR_F_KSG_DENSE: eps / counts bit-exact,
    sweep == dense bit for bit."""
    n = 1000
    sa = synth.field_spec(4, 4, 2, n, seed=11)
    sb = synth.field_spec(4, 4, 2, n, seed=12, variable=2)
    va, fa = _field(sa)
    vb, fb = _field(sb)
    a, b = synth.random_pairs(sa.points, 24, seed=k)
    a, b = a.numpy(), b.numpy()
    _check_knn(fa, va, k, a, b, fb=fb, vals_b=vb)
    ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    got = _cpu(cb.corr_eval_pairs(fa, fb, cb.CORR_KSG, k, ta, tb))
    dense = _cpu(cb.corr_eval_pairs(fa, fb, cb.CORR_KSG | cb.CORR_F_KSG_DENSE, k, ta, tb))
    ref = oracle.eval_pairs(va.cpu(), vb.cpu(), oracle.KSG, k, a, b)
    assert np.array_equal(got, dense, equal_nan=True)
    assert np.max(np.abs(got - ref)) <= KSG_TOL
    fa.close()
    fb.close()


def test_pearson_screen_many_near_max_tiles():
    """The exhaustive Pearson path screens tiles with the hi*hi product and runs the exact split-TF32
    product only where a tile can hold the region pair's maximum.  Here every series is one shared
    signal plus small noise (|r| ~ 0.999 everywhere), so nearly all tiles lie within the screening
    margin and pass 2 runs on a long tile list; half of the B points carry the negated signal
    (CORR_F_ABS), and two B points duplicate A points exactly (r = 1 up to rounding)."""
    n, nx, ny, nz = 100, 64, 32, 4
    g = torch.Generator().manual_seed(21)
    sig = torch.randn(n, 1, generator=g, dtype=torch.float64)
    noise = torch.randn(n, nx * ny * nz, generator=g, dtype=torch.float64)
    vals = (sig + 0.03 * noise).to(torch.float32)
    vals[:, nx // 2 + 8::nx] *= -1  # a column of B with the negated signal
    p_a1, p_a2 = 5 * nx + 3, 17 * nx + 30                     # in A = x < 32
    p_b1, p_b2 = 9 * nx + 40, 2 * nx * ny + 20 * nx + 50     # in B = x >= 32
    vals[:, p_b1] = vals[:, p_a1]
    vals[:, p_b2] = vals[:, p_a2]
    f = cb.corr_field_create(vals.cuda(), nx, ny, nz, n)
    host = vals.numpy()
    A, B = [(0, 0, 0, 32, ny, nz)], [(32, 0, 0, nx, ny, nz)]
    _block_compare(f, None, host, None, (nx, ny, nz), A, B)
    _block_compare(f, None, host, None, (nx, ny, nz), A, B, absval=True)
    m, a = cb.corr_region_max(f, None, cb.CORR_PEARSON, 0, A, B, 0, 0)
    # the two duplicated series give r = 1 up to the split-TF32 rounding (~1e-6): one of them wins
    assert abs(float(m[0]) - 1.0) <= PEARSON_TOL and tuple(_cpu(a)[0]) in ((p_a1, p_b1), (p_a2, p_b2))
    f.close()


@pytest.mark.parametrize("n", [100, 1000])
def test_batch_equals_single_calls(n):
    """a batch of point pairs gives bit-for-bit the results of one call per pair
    (pairs are independent units; the sampler and the schedule never mix them)."""
    spec = synth.field_spec(8, 8, 2, n, seed=31 + n)
    vals, f = _field(spec)
    a, b = synth.random_pairs(spec.points, 24, seed=n)
    ta, tb = a.cuda(), b.cuda()
    for measure in (cb.CORR_KSG, cb.CORR_PEARSON, cb.CORR_KSG | cb.CORR_F_KSG_PLUS1):
        batch = _cpu(cb.corr_eval_pairs(f, None, measure, 3, ta, tb))
        single = np.concatenate([_cpu(cb.corr_eval_pairs(f, None, measure, 3, ta[i:i + 1], tb[i:i + 1]))
                                 for i in range(len(a))])
        assert np.array_equal(batch, single, equal_nan=True), measure
    f.close()


@pytest.mark.parametrize("n,k,npairs", [(2000, 0, 10), (4096, 0, 3), (1000, 33, 12), (1000, 64, 10),
                                        (100, 50, 40), (100, 99, 40), (300, 200, 8), (130, 97, 16)])
def test_large_k_multipass(n, k, npairs):
    """k >= 33 (the paper's k = ceil(3n/100) for n >= 1067: 60 at n = 2000, 123 at n = 4096;
    PAPER.md:173) runs the multi-pass batched lists: eps / counts bit-exact vs the oracle, MI
    within 1e-4, and the pruned and dense passes bit-identical (incl. k = n - 1)."""
    spec = synth.field_spec(4, 4, 2, n, seed=3 * n + k)
    vals, f = _field(spec)
    a, b = synth.random_pairs(spec.points, npairs, seed=n + k)
    a, b = a.numpy(), b.numpy()
    kk = k if k else min(max(1, -(-3 * n // 100)), n - 1)
    assert kk >= 33
    _check_knn(f, vals, kk, a, b)
    ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    got = _cpu(cb.corr_eval_pairs(f, None, cb.CORR_KSG, k, ta, tb))
    dense = _cpu(cb.corr_eval_pairs(f, None, cb.CORR_KSG | cb.CORR_F_KSG_DENSE, k, ta, tb))
    ref = oracle.eval_pairs(vals.cpu(), None, oracle.KSG, kk, a, b)
    assert np.array_equal(got, dense, equal_nan=True)
    assert np.array_equal(np.isnan(got), np.isnan(ref))
    ok = ~np.isnan(ref)
    assert np.max(np.abs(got[ok] - ref[ok]), initial=0) <= KSG_TOL
    f.close()


@pytest.mark.parametrize("k", [33, 64, 100])
def test_large_k_multipass_ties(k):
    """Heavily quantised series (many equal distances at every pass's floor): the multi-pass
    lists must count the floor's tie copies exactly (eps may equal the floor value)."""
    n, P = 200, 64
    g = torch.Generator().manual_seed(k)
    vals = (torch.randint(0, 6, (n, P), generator=g).to(torch.float32) * 0.5).contiguous()
    f = cb.corr_field_create(vals.cuda(), 8, 8, 1, n)
    a, b = synth.random_pairs(P, 60, seed=k)
    _check_knn(f, vals, k, a.numpy(), b.numpy())
    f.close()


@pytest.mark.parametrize("n", [100, 300])
def test_ksg_nan_pairs_counted(n):
    """Zero-inflated series (R5: duplicate joint samples -> eps = 0 -> psi(0) -> NaN) and constant
    series (R10): corr_region_max skips their NaN values, and corr_ksg_nan_pairs reports exactly
    the number of skipped sampled pairs the oracle's enumeration finds NaN (warp kernel at n = 100,
    column-cell kernel at n = 300)."""
    nx, ny, nz = 8, 8, 2
    g = torch.Generator().manual_seed(n)
    vals = torch.rand((n, nx * ny * nz), generator=g)
    vals[torch.rand(vals.shape, generator=g) < 0.4] = 0.0
    vals[:, 5] = 1.5  # a constant series
    vals = vals.contiguous()
    f = cb.corr_field_create(vals.cuda(), nx, ny, nz, n)
    boxes = synth.partition(nx, ny, nz, 4, 4, 2)
    A, B = synth.context_pairs(boxes)
    S = 64
    cb.corr_ksg_nan_pairs(0, reset=True)
    gm, ga = cb.corr_region_max(f, None, cb.CORR_KSG, 3, A, B, S, 5)
    got = cb.corr_ksg_nan_pairs(0, reset=True)
    vals_o, va, vb = oracle.region_values(vals, None, (nx, ny, nz), oracle.KSG, 3, A, B, S, 5)
    assert got == int(np.isnan(vals_o).sum()) and got > 0
    mx, arg, sec, value_at = oracle_region_reference(vals, None, (nx, ny, nz), oracle.KSG, 3, A, B, S, 5)
    assert_region_argmax(_cpu(gm), _cpu(ga), mx, arg, sec, KSG_TOL, value_at)
    f.close()


def test_concurrent_streams_same_field():
    """The field is immutable after creation (corr.h): region-max calls on two streams at once
    (sharing the resident region table and its events) give the results of sequential calls."""
    spec = synth.spec_of(synth.C3)
    vals, f = _field(spec)
    del vals
    A, B = synth.context_pairs(synth.bricks_of(synth.C3))
    A, B = A[:600], B[:600]
    ref_k = cb.corr_region_max(f, None, cb.CORR_KSG, 3, A, B, 64, 3)
    ref_p = cb.corr_region_max(f, None, cb.CORR_PEARSON, 0, A, B, 64, 4)
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(3):
        with torch.cuda.stream(s1):
            got_k = cb.corr_region_max(f, None, cb.CORR_KSG, 3, A, B, 64, 3, stream=s1)
        with torch.cuda.stream(s2):
            got_p = cb.corr_region_max(f, None, cb.CORR_PEARSON, 0, A, B, 64, 4, stream=s2)
        torch.cuda.synchronize()
        assert torch.equal(got_k[0], ref_k[0]) and torch.equal(got_k[1], ref_k[1])
        assert torch.equal(got_p[0], ref_p[0]) and torch.equal(got_p[1], ref_p[1])
    f.close()


_QUEUE_SCRIPT = r"""
import sys
import numpy as np
import torch
sys.path[:0] = [{root!r}, {tests!r}]
import oracle
from paper_2309_03308_b200 import binding as cb
from paper_2309_03308_b200 import synth
spec = synth.field_spec(8, 8, 4, 1000, seed=4242)
vals = synth.generate(spec, device="cuda")
f = cb.corr_field_create(vals, spec.nx, spec.ny, spec.nz, spec.members)
a, b = synth.random_pairs(spec.points, 48, seed=7)
a, b = a.numpy(), b.numpy()
eps, nx, ny = cb.corr_ksg_debug(f, None, 3, torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda())
cb.corr_check(f)
reps, rnx, rny = oracle.knn_pairs(vals.cpu(), None, 3, a, b)
ok = (np.array_equal(eps.cpu().numpy(), reps) and np.array_equal(nx.cpu().numpy(), rnx)
      and np.array_equal(ny.cpu().numpy(), rny))
print("bit-exact" if ok else "MISMATCH")
sys.exit(0 if ok else 1)
"""


@pytest.mark.parametrize("qcap", ["0", "2", "128"])
def test_ksg_far_visit_queue_capacities(qcap):
    """The column-cell kernel's far-visit queue: no queue (every far visit in the
    column warp), a 2-entry queue (almost every far lane overflows back into its column warp) and
    the default capacity give bit-exact eps / counts at n = 1000.  The capacity is read once per
    process (CORR_KSG_QUEUE), hence the subprocess."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = _QUEUE_SCRIPT.format(root=root, tests=os.path.join(root, "tests"))
    env = dict(os.environ, CORR_KSG_QUEUE=qcap)
    r = subprocess.run([sys.executable, "-c", script], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "bit-exact" in r.stdout, r.stdout + r.stderr


_SCREEN_SCRIPT = r"""
import sys
import numpy as np
sys.path[:0] = [{root!r}]
from paper_2309_03308_b200 import binding as cb
from paper_2309_03308_b200 import synth
spec = synth.spec_of(synth.C3)
vals = synth.generate(spec, device="cuda")
f = cb.corr_field_create(vals, spec.nx, spec.ny, spec.nz, spec.members)
bricks = synth.bricks_of(synth.C3)
A = [bricks[7], bricks[0], (0, 0, 0, 16, 8, 3), (100, 100, 3, 164, 110, 9)]
B = [bricks[80], bricks[87], (4, 2, 0, 12, 10, 4), (120, 96, 0, 150, 140, 20)]
m, a = cb.corr_region_max(f, None, cb.CORR_PEARSON, 0, A, B, 0, 0)
np.save(sys.argv[1], np.concatenate([m.cpu().numpy().view(np.int32).astype(np.int64), a.cpu().numpy().ravel()]))
"""


def test_pearson_screen_multicast_equals_single_sm(tmp_path):
    """The multicast bf16 screen (default) and the 1-SM screen (CORR_GEMM_SCREEN_MC=0) select
    tiles from bit-identical screening values, so the exhaustive maxima and argmaxes agree bit for
    bit (boundary, odd-tile and overlapping boxes)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = _SCREEN_SCRIPT.format(root=root)
    outs = []
    for mc in ("1", "0"):
        path = str(tmp_path / f"mc{mc}.npy")
        env = dict(os.environ, CORR_GEMM_SCREEN_MC=mc)
        r = subprocess.run([sys.executable, "-c", script, path], env=env, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stdout + r.stderr
        outs.append(np.load(path))
    assert np.array_equal(outs[0], outs[1])
