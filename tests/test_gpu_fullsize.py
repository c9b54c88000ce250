"""GPU parity at the BASELINE.json configs' FULL sizes (C2-C5), in the launch configurations the
bench times, against the CPU oracle ("Next round" item 1).

The oracle cannot evaluate every one of 4.2e8 (C2) or 3.1e12 (C5) point pairs, so each check is
chosen so that a wrong GPU result anywhere it looks fails it:
  * element by element on large random subsets (eps / counts bit-exact, MI <= 1e-4);
  * the region argmax of EVERY region pair is one of that region's candidates (sampler re-derived
    by the oracle) and its oracle value equals the GPU maximum within the tolerance;
  * full enumerations of some region pairs with the argmax-margin rule (argmax bit-exact whenever
    the oracle's winning margin exceeds the tolerance, tests/parity_helpers.py);
  * C3 S = 100 (the paper's BOS budget): every sample of all 3828 region pairs.
Rows are regenerated on the host by the shared input generator (synth.rows), never read back
from the CUDA path.
"""
import numpy as np
import pytest
import torch

import oracle
from paper_2309_03308_b200 import binding as cb
from paper_2309_03308_b200 import synth
from parity_helpers import assert_region_argmax, enumerated_value_at, in_box, oracle_region_reference

pytestmark = pytest.mark.gpu

KSG_TOL = 1e-4
PEARSON_TOL = 1e-5
BENCH_SEED = 20230907  # bench.py SEED


def _field(spec):
    vals = synth.generate(spec, device="cuda")
    f = cb.corr_field_create(vals, spec.nx, spec.ny, spec.nz, spec.members)
    return vals, f


def _box_points(box, nx, ny):
    x0, y0, z0, x1, y1, z1 = box
    z, y, x = np.meshgrid(np.arange(z0, z1), np.arange(y0, y1), np.arange(x0, x1), indexing="ij")
    return ((z * ny + y) * nx + x).reshape(-1).astype(np.int64)


class Rows:
    """Host rows of a set of grid points (shared generator), as an oracle field [n, m] plus the
    map global point -> column.  Two-field oracle calls need both Rows built on the SAME point
    set (the oracle indexes both fields with one point count)."""

    def __init__(self, spec, points):
        self.pts = np.unique(np.asarray(points, np.int64))
        self.pos = {int(p): i for i, p in enumerate(self.pts)}
        self.vals = synth.rows(spec, torch.from_numpy(self.pts)).T.contiguous().numpy()

    def idx(self, p):
        return np.searchsorted(self.pts, np.asarray(p, np.int64))


def _oracle_at(measure, k, ra, rb, a, b):
    """Oracle values (rounded to the library's fp32) of global pairs (a, b); rb None = one field."""
    if rb is None:
        v = oracle.eval_pairs(ra.vals, None, measure, k, ra.idx(a), ra.idx(b))
    else:
        v = oracle.eval_pairs(ra.vals, rb.vals, measure, k, ra.idx(a), rb.idx(b))
    v = v.astype(np.float32).astype(np.float64)
    return np.abs(v) if measure & oracle.F_ABS else v


def test_c2_ksg_exhaustive_focus():
    """C2: KSG (k = 3) over ALL 4.19e8 point pairs of the two focus bricks (n = 100).  1e5 random
    pairs of the 4.19e8: eps / counts bit-exact, MI within 1e-4; the GPU argmax pair recomputed
    by the oracle equals the GPU max; no oracle-evaluated pair exceeds the max + 1e-4."""
    spec = synth.spec_of(synth.C2)
    vals, f = _field(spec)
    del vals
    A, B = synth.C2_REGION_A, synth.C2_REGION_B
    gm, ga = cb.corr_region_max(f, None, cb.CORR_KSG, 3, [A], [B], 0, 0)
    gm, ga = float(gm.cpu()[0]), tuple(int(v) for v in ga.cpu()[0])
    pa, pb = _box_points(A, spec.nx, spec.ny), _box_points(B, spec.nx, spec.ny)
    rows = Rows(spec, np.concatenate([pa, pb]))
    rng = np.random.default_rng(2)
    a = pa[rng.integers(0, pa.size, 100_000)]
    b = pb[rng.integers(0, pb.size, 100_000)]
    ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    got = cb.corr_eval_pairs(f, None, cb.CORR_KSG, 3, ta, tb).cpu().numpy().astype(np.float64)
    ref = _oracle_at(oracle.KSG, 3, rows, None, a, b)
    assert np.array_equal(np.isnan(got), np.isnan(ref))
    ok = ~np.isnan(ref)
    assert np.max(np.abs(got[ok] - ref[ok])) <= KSG_TOL
    eps, nx, ny = cb.corr_ksg_debug(f, None, 3, ta, tb)
    reps, rnx, rny = oracle.knn_pairs(rows.vals, None, 3, rows.idx(a), rows.idx(b))
    assert np.array_equal(eps.cpu().numpy(), reps)
    assert np.array_equal(nx.cpu().numpy(), rnx) and np.array_equal(ny.cpu().numpy(), rny)
    del eps, nx, ny
    # the exhaustive maximum covers every evaluated pair, bit for bit (same kernel arithmetic)
    assert np.nanmax(got) <= gm
    assert in_box(ga[0], A, spec.nx, spec.ny) and in_box(ga[1], B, spec.nx, spec.ny)
    v_arg = _oracle_at(oracle.KSG, 3, rows, None, [ga[0]], [ga[1]])[0]
    assert abs(v_arg - gm) <= KSG_TOL, (v_arg, gm)
    assert np.nanmax(ref) <= gm + KSG_TOL
    cb.corr_check(f)
    f.close()


@pytest.mark.parametrize("measure,tol", [(cb.CORR_KSG, KSG_TOL), (cb.CORR_PEARSON, PEARSON_TOL)])
def test_c3_s100_all_region_pairs_full(measure, tol):
    """C3 (n = 100), S = 100 samples (the paper's BOS budget) for all 3828 region pairs: every one
    of the 382 800 sampled pairs evaluated by the oracle; max within tol, argmax-margin rule."""
    spec = synth.spec_of(synth.C3)
    vals, f = _field(spec)
    host = vals.cpu()
    del vals
    A, B = synth.context_pairs(synth.bricks_of(synth.C3))
    gm, ga = cb.corr_region_max(f, None, measure, 3, A, B, 100, 777)
    mx, arg, sec, value_at = oracle_region_reference(host, None, (spec.nx, spec.ny, spec.nz), measure, 3, A, B,
                                                     100, 777)
    assert_region_argmax(gm.cpu().numpy(), ga.cpu().numpy(), mx, arg, sec, tol, value_at)
    f.close()


def _check_all_argmax(spec_a, spec_b, fa, fb, measure, k, A, B, S, seed, tol, full_regions, nprobe):
    """For EVERY region pair: the GPU argmax is one of its S sampled pairs and its oracle value
    equals the GPU max within tol.  For `full_regions`: all S samples by the oracle, margin rule.
    Random probes: no sampled pair's oracle value exceeds the GPU max + tol."""
    nx, ny = spec_a.nx, spec_a.ny
    gm, ga = cb.corr_region_max(fa, fb, measure, k, A, B, S, seed)
    gm, ga = gm.cpu().numpy().astype(np.float64), ga.cpu().numpy()
    sa, sb = oracle.sample_many(seed, A, B, S, nx, ny)
    member = ((sa == ga[:, :1]) & (sb == ga[:, 1:])).any(axis=1)
    assert member.all(), np.nonzero(~member)[0][:10]
    rng = np.random.default_rng(5)
    probe_r = rng.integers(0, len(A), nprobe)
    probe_s = rng.integers(0, S, nprobe)
    pa = np.concatenate([ga[:, 0], sa[full_regions].reshape(-1), sa[probe_r, probe_s]])
    pb = np.concatenate([ga[:, 1], sb[full_regions].reshape(-1), sb[probe_r, probe_s]])
    ra = Rows(spec_a, np.concatenate([pa, pb]))
    rb = None if spec_b is None else Rows(spec_b, np.concatenate([pa, pb]))  # same columns as ra
    v = _oracle_at(measure, k, ra, rb, pa, pb)
    R = len(A)
    v_arg = v[:R]
    assert np.all(np.abs(v_arg - gm) <= tol), np.max(np.abs(v_arg - gm))
    nf = len(full_regions) * S
    vals = v[R:R + nf].reshape(len(full_regions), S)
    mx, arg, sec = oracle.select_max(vals, sa[full_regions], sb[full_regions])
    assert_region_argmax(gm[full_regions], ga[full_regions], mx, arg, sec, tol,
                         enumerated_value_at(vals, sa[full_regions], sb[full_regions]))
    vp = v[R + nf:]
    assert np.all(np.isnan(vp) | (vp <= gm[probe_r] + tol))


@pytest.mark.parametrize("measure,tol,full,nprobe", [(cb.CORR_KSG, KSG_TOL, [1234], 1024),
                                                     (cb.CORR_PEARSON, PEARSON_TOL, [0, 77, 1234, 3827], 20000)])
def test_c4_bench_launch_all_region_pairs(measure, tol, full, nprobe):
    """The bench's exact launch: C4 (n = 1000), all 3828 region pairs, S = 4096, bench seed."""
    spec = synth.spec_of(synth.C4)
    vals, f = _field(spec)
    del vals
    torch.cuda.empty_cache()
    A, B = synth.context_pairs(synth.bricks_of(synth.C4))
    _check_all_argmax(spec, None, f, None, measure, 3, A, B, 4096, BENCH_SEED, tol, full, nprobe)
    f.close()


@pytest.fixture(scope="module")
def c5_fields():
    sa, sb = synth.spec_of(synth.C5, 1), synth.spec_of(synth.C5, 2)
    va, fa = _field(sa)
    del va
    vb, fb = _field(sb)
    del vb
    torch.cuda.empty_cache()
    yield sa, sb, fa, fb
    fa.close()
    fb.close()
    torch.cuda.empty_cache()


def test_c5_ksg_s1024_all_region_pairs(c5_fields):
    """C5 (two fields, n = 1000): KSG S = 1024 over all 7744 ordered region pairs."""
    sa, sb, fa, fb = c5_fields
    A, B = synth.matrix_pairs(synth.bricks_of(synth.C5))
    _check_all_argmax(sa, sb, fa, fb, cb.CORR_KSG, 3, A, B, 1024, BENCH_SEED, KSG_TOL, [4000], 512)


def test_c5_pearson_exhaustive_matrix(c5_fields):
    """C5: Pearson over ALL 3.1e12 point pairs of the 7744 ordered brick pairs.  Every argmax lies
    in its boxes and its oracle value equals the GPU max; 4 brick pairs are recomputed in full by
    the oracle's fp64 block max (incl. the boundary bricks and the matrix maximum's pair) with the
    argmax-margin rule."""
    sa, sb, fa, fb = c5_fields
    bricks = synth.bricks_of(synth.C5)
    A, B = synth.matrix_pairs(bricks)
    gm, ga = cb.corr_region_max(fa, fb, cb.CORR_PEARSON, 0, A, B, 0, 0)
    gm, ga = gm.cpu().numpy().astype(np.float64), ga.cpu().numpy()
    for r in range(len(A)):
        assert in_box(ga[r][0], A[r], sa.nx, sa.ny) and in_box(ga[r][1], B[r], sa.nx, sa.ny), r
    ra, rb = Rows(sa, ga.reshape(-1)), Rows(sb, ga.reshape(-1))  # same columns (the oracle's P)
    v = _oracle_at(oracle.PEARSON, 0, ra, rb, ga[:, 0], ga[:, 1])
    assert np.all(np.abs(v - gm) <= PEARSON_TOL), np.max(np.abs(v - gm))
    top = int(np.nanargmax(gm))
    for r in sorted({top, 7, 88 * 7 + 80, len(A) - 1}):
        pa, pb = _box_points(A[r], sa.nx, sa.ny), _box_points(B[r], sa.nx, sa.ny)
        xa = synth.rows(sa, torch.from_numpy(pa)).T.contiguous().numpy()
        xb = synth.rows(sb, torch.from_numpy(pb)).T.contiguous().numpy()
        # the two bricks as their own grids: local index = position in _box_points order
        mx, ab, sec = _block_max_two_grids(xa, xb)
        ref_arg = (int(pa[ab[0]]), int(pb[ab[1]]))

        def value_at(_r, g):
            if not (in_box(g[0], A[r], sa.nx, sa.ny) and in_box(g[1], B[r], sa.nx, sa.ny)):
                return None
            w = _oracle_at(oracle.PEARSON, 0, Rows(sa, [g[0]]), Rows(sb, [g[1]]), [g[0]], [g[1]])[0]
            return None if np.isnan(w) else float(w)

        assert_region_argmax(gm[r:r + 1], ga[r:r + 1], np.array([mx]), np.array([ref_arg]), np.array([sec]),
                             PEARSON_TOL, lambda _i, g: value_at(r, g))


def _block_max_two_grids(xa, xb):
    """oracle.pearson_block_max over two bricks given as their own fields ([n, |A|], [n, |B|]); the
    concatenation trick: one grid of |A| + |B| points laid out along x, A = first |A|, B = rest."""
    na, nb = xa.shape[1], xb.shape[1]
    both = np.concatenate([xa, xb], axis=1)
    dims = (na + nb, 1, 1)
    mx, ab, sec = oracle.pearson_block_max(both, None, dims, (0, 0, 0, na, 1, 1), (na, 0, 0, na + nb, 1, 1),
                                           runner_up=True)
    return mx, (ab[0], ab[1] - na), sec


def test_c4_paper_k_rule_all_region_pairs():
    """C4 with the paper's k = ceil(3n/100) = 30 (k = 0; batched 32-entry lists),
    S = 64, all 3828 region pairs: every argmax is a sampled pair whose oracle value equals the GPU
    max; one region pair enumerated in full with the margin rule."""
    spec = synth.spec_of(synth.C4)
    vals, f = _field(spec)
    del vals
    torch.cuda.empty_cache()
    A, B = synth.context_pairs(synth.bricks_of(synth.C4))
    k = -(-3 * spec.members // 100)
    assert k == 30
    m0, a0 = cb.corr_region_max(f, None, cb.CORR_KSG, 0, A, B, 64, BENCH_SEED)   # k = 0: the rule
    m1, a1 = cb.corr_region_max(f, None, cb.CORR_KSG, k, A, B, 64, BENCH_SEED)
    assert torch.equal(m0, m1) and torch.equal(a0, a1)
    _check_all_argmax(spec, None, f, None, cb.CORR_KSG, k, A, B, 64, BENCH_SEED, KSG_TOL, [2000], 256)
    f.close()
