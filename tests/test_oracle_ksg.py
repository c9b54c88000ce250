"""Pins for the oracle's Chebyshev k-NN, marginal counts and KSG MI (CPU only).

Definitions: PAPER.md:172-174 (§3.2).  Readings R1-R7 of DESIGN.md.
Pins, each chosen so that a plausible bug (wrong k index, non-strict count,
missing self-exclusion, dropped psi term, wrong sign) fails one of them:

* SPEC worked example (golden) and the k = n-1 special case;
* scipy.spatial.cKDTree(p=inf): fp32 rounding is monotone, so the k-th smallest
  fp32 distance equals fp32(k-th smallest exact distance) -- bit-exact;
* an independent count algorithm (sorted marginal + monotone predicate scan);
* order-statistic properties of eps and the k-1 lower bound of the counts;
* closed forms: the self pair y = x gives psi(n)+psi(k)-2psi(k-1) (verbatim) and
  psi(n)-psi(k) (+1 variant), via scipy.special.digamma; the bivariate Gaussian
  -1/2 ln(1-rho^2) for the +1 variant at n = 1000;
* exact identity verbatim - plus1 = (1/n) sum (1/n_x + 1/n_y);
* bit-exact invariances (swap, reflection, power-of-two scale, permutation,
  rank transform of a monotone map);
* degenerate cases: constant series and psi(0) -> NaN.
"""
import concurrent.futures as cf
import math

import numpy as np
import pytest
import scipy.special
from scipy.spatial import cKDTree

import oracle
from conftest import read_golden


def _data(n, seed, rho=0.0):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal(n)
    y = rho * x + math.sqrt(1 - rho * rho) * rng.standard_normal(n)
    return x.astype(np.float32), y.astype(np.float32)


def _temperature_like(n, seed):
    """fp32 values with many exact ties, like the generator's fields."""
    rng = np.random.default_rng(seed)
    x = (250.0 + 0.5 * rng.standard_normal(n)).astype(np.float32)
    y = (255.0 + 1.5 * rng.standard_normal(n)).astype(np.float32)
    return x, y


def test_knn_spec_example():
    row = read_golden("knn_spec_example.txt")[0]
    x = [float(v) for v in row[0].split()]
    y = [float(v) for v in row[1].split()]
    eps, nx, ny = oracle.knn(x, y, int(row[2]))
    assert eps.tolist() == [float(v) for v in row[3].split()]
    assert nx.tolist() == [int(v) for v in row[4].split()]
    assert ny.tolist() == [int(v) for v in row[5].split()]


def test_knn_k_equals_n_minus_1_is_farthest():
    x, y = _data(50, 1)
    eps, _, _ = oracle.knn(x, y, 49)
    for i in range(50):
        far = max(max(abs(np.float32(x[i] - x[j])), abs(np.float32(y[i] - y[j])))
                  for j in range(50) if j != i)
        assert eps[i] == far


@pytest.mark.parametrize("n,k,seed,kind", [(10, 3, 1, "normal"), (100, 3, 2, "normal"),
                                           (257, 7, 3, "normal"), (1000, 3, 4, "normal"),
                                           (300, 3, 5, "temp"), (100, 1, 6, "normal"),
                                           (200, 30, 7, "temp")])
def test_eps_equals_kdtree_rounded(n, k, seed, kind):
    x, y = _data(n, seed) if kind == "normal" else _temperature_like(n, seed)
    eps, _, _ = oracle.knn(x, y, k)
    pts = np.stack([x.astype(np.float64), y.astype(np.float64)], axis=1)
    d, _ = cKDTree(pts).query(pts, k=k + 1, p=np.inf)
    kd = d[:, k].astype(np.float32)  # self is the 0-th neighbour (distance 0)
    assert np.array_equal(eps, kd)


def _count_sorted(v, eps):
    """Independent algorithm: scan the sorted marginal with a monotone predicate."""
    s = np.sort(v)
    out = np.empty(v.size, np.int64)
    for i in range(v.size):
        xi, e = v[i], eps[i]
        up = (s >= xi) & (np.abs(s - xi) >= e)          # monotone F..FT..T
        lo = (s >= xi) | (np.abs(xi - s) < e)           # monotone F..FT..T
        u = int(np.argmax(up)) if up.any() else s.size
        w = int(np.argmax(lo)) if lo.any() else s.size
        out[i] = (u - w) - (1 if e > 0 else 0)
    return out


@pytest.mark.parametrize("n,k,seed,kind", [(100, 3, 8, "normal"), (500, 3, 9, "temp"),
                                           (300, 5, 10, "normal")])
def test_counts_independent_sorted_algorithm(n, k, seed, kind):
    x, y = _data(n, seed, 0.6) if kind == "normal" else _temperature_like(n, seed)
    eps, nx, ny = oracle.knn(x, y, k)
    assert np.array_equal(nx, _count_sorted(x, eps))
    assert np.array_equal(ny, _count_sorted(y, eps))


def test_eps_order_statistic_and_count_bounds():
    for n, k, seed in ((100, 3, 20), (400, 4, 21), (64, 1, 22)):
        x, y = _data(n, seed, 0.3)
        eps, nx, ny = oracle.knn(x, y, k)
        D = np.maximum(np.abs(x[:, None] - x[None, :]), np.abs(y[:, None] - y[None, :]))
        np.fill_diagonal(D, np.inf)
        for i in range(n):
            row = D[i][np.isfinite(D[i])]
            assert (row < eps[i]).sum() <= k - 1
            assert (row <= eps[i]).sum() >= k
            assert eps[i] in row
            if (row == eps[i]).sum() == 1:  # no tie at rank k
                assert nx[i] >= k - 1 and ny[i] >= k - 1


def _psi(m):
    return float(scipy.special.digamma(m))


@pytest.mark.parametrize("n", [10, 100, 1000])
def test_ksg_self_pair_closed_form(n):
    rng = np.random.default_rng(n)
    x = rng.permutation(np.arange(n, dtype=np.float64) ** 1.5 + rng.random(n) * 0.01)
    x = x.astype(np.float32)
    k = 3
    gaps = np.abs(x[:, None] - x[None, :])
    np.fill_diagonal(gaps, np.inf)
    srt = np.sort(gaps, axis=1)
    assert (srt[:, k - 2] < srt[:, k - 1]).all()  # no tie between ranks k-1 and k in any row
    assert oracle.ksg(x, x, k) == pytest.approx(_psi(n) + _psi(k) - 2 * _psi(k - 1), abs=1e-12)
    assert oracle.ksg(x, x, k, plus1=True) == pytest.approx(_psi(n) - _psi(k), abs=1e-12)


def test_ksg_bounds():
    for seed in range(5):
        x, y = _data(200, 100 + seed, 0.5)
        k, n = 3, 200
        v = oracle.ksg(x, y, k)
        assert v <= _psi(n) + _psi(k) - 2 * _psi(k - 1) + 1e-12
        assert v >= _psi(n) + _psi(k) - 2 * _psi(n - 1) - 1e-12


def test_ksg_verbatim_plus1_identity():
    for seed in range(4):
        x, y = _data(300, 200 + seed, 0.7)
        _, nx, ny = oracle.knn(x, y, 3)
        diff = oracle.ksg(x, y, 3) - oracle.ksg(x, y, 3, plus1=True)
        assert diff == pytest.approx(np.mean(1.0 / nx + 1.0 / ny), abs=1e-12)


def test_ksg_gaussian_closed_form():
    """20-seed mean within 0.05 nats of -1/2 ln(1-rho^2), n=1000 (+1 form)."""
    jobs = [(rho, s) for rho in (0.0, 0.5, 0.9) for s in range(20)]

    def one(job):
        rho, s = job
        x, y = _data(1000, 1000 * s + int(rho * 10), rho)
        return rho, oracle.ksg(x, y, 3, plus1=True)

    with cf.ThreadPoolExecutor(8) as ex:
        res = list(ex.map(one, jobs))
    for rho in (0.0, 0.5, 0.9):
        vals = [v for r, v in res if r == rho]
        truth = -0.5 * math.log(1 - rho * rho)
        assert abs(np.mean(vals) - truth) <= 0.05, (rho, np.mean(vals), truth)
        if rho == 0.0:
            assert abs(np.mean(vals)) <= 0.02


def test_ksg_bit_exact_invariances():
    x, y = _temperature_like(300, 31)
    k = 3
    base = oracle.ksg(x, y, k)
    assert oracle.ksg(y, x, k) == base                               # swap (Eq. 1 symmetry)
    assert oracle.ksg(-x, y, k) == base                              # reflection
    assert oracle.ksg(np.float32(4.0) * x, np.float32(4.0) * y, k) == base  # common 2^m scale
    perm = np.random.default_rng(3).permutation(300)
    assert oracle.ksg(x[perm], y[perm], k) == base                   # member permutation


def test_ksg_rank_transform_monotone_invariance():
    x, y = _data(400, 41, 0.6)
    rx = np.argsort(np.argsort(x)).astype(np.float32)
    ry = np.argsort(np.argsort(y)).astype(np.float32)
    fx = np.argsort(np.argsort(x.astype(np.float64) ** 3 + 5 * x)).astype(np.float32)
    assert oracle.ksg(rx, ry, 3) == oracle.ksg(fx, ry, 3)


def test_ksg_degenerate_nan():
    x, _ = _data(100, 51)
    assert math.isnan(oracle.ksg(np.full(100, 3.0, np.float32), x, 3))
    assert math.isnan(oracle.ksg(x, np.full(100, -1.0, np.float32), 3))
    rng = np.random.default_rng(52)
    z = np.where(rng.random(200) < 0.6, 0.0, rng.random(200)).astype(np.float32)
    w = np.where(rng.random(200) < 0.6, 0.0, rng.random(200)).astype(np.float32)
    eps, nx, ny = oracle.knn(z, w, 3)
    assert (eps == 0).any() and (nx[eps == 0] == 0).all() and (ny[eps == 0] == 0).all()
    assert math.isnan(oracle.ksg(z, w, 3))                 # psi(0) in the verbatim form
    assert math.isfinite(oracle.ksg(z, w, 3, plus1=True))  # +1 form stays finite
