"""Pins for the oracle's sampler (R15) and region-pair maximum.

* mix64: the published splitmix64 seed-0 output sequence (golden);
* sampled points lie in their boxes and are uniform (chi-square);
* the key depends only on (seed, boxes): a shard of the region list draws the
  same samples as the full list (determinism across 1..8 GPUs);
* region max equals the max over the explicitly evaluated pair list, with NaN
  skipped, lowest-index ties and self pairs excluded;
* closed form: generator cluster centres share one signal, so series at two
  centres are affine-related and their PPMCC region max is 1.
"""
import numpy as np
import pytest
import torch

import oracle
from conftest import read_golden
from paper_2309_03308_b200 import synth


def test_mix64_splitmix_vectors():
    vals = [int(r[0], 16) for r in read_golden("splitmix64_vectors.txt")]
    state = 0
    for v in vals:
        state = (state + 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF
        assert oracle.mix64(state) == v


def test_samples_in_box_and_uniform():
    nx, ny, nz = 250, 352, 20
    A = (32, 64, 0, 64, 96, 20)
    B = (218, 320, 0, 250, 352, 20)
    cnt = np.zeros(synth.box_size(A), np.int64)
    for s in range(20000):
        a, b = oracle.sample(7, A, B, s, nx, ny)
        ax, ay, az = a % nx, (a // nx) % ny, a // (nx * ny)
        bx, by, bz = b % nx, (b // nx) % ny, b // (nx * ny)
        assert A[0] <= ax < A[3] and A[1] <= ay < A[4] and A[2] <= az < A[5]
        assert B[0] <= bx < B[3] and B[1] <= by < B[4] and B[2] <= bz < B[5]
        cnt[(az - A[2]) * 32 * 32 + (ay - A[1]) * 32 + (ax - A[0])] += 1
    # chi-square over 64 coarse bins of the A-local index
    coarse = cnt.reshape(64, -1).sum(1)
    exp = coarse.sum() / 64
    chi2 = ((coarse - exp) ** 2 / exp).sum()
    assert chi2 < 120  # 63 dof, p ~ 1e-5


def test_sample_key_depends_only_on_boxes():
    A, B = (0, 0, 0, 4, 4, 4), (4, 4, 0, 8, 8, 4)
    assert oracle.pair_key(5, A, B) == oracle.pair_key(5, A, B)
    assert oracle.pair_key(5, A, B) != oracle.pair_key(5, B, A)
    assert oracle.pair_key(5, A, B) != oracle.pair_key(6, A, B)


def _c1_field():
    spec = synth.spec_of(synth.C1)
    return spec, synth.generate(spec).numpy()


@pytest.mark.parametrize("measure", [oracle.PEARSON, oracle.KSG, oracle.KSG | oracle.F_KSG_PLUS1,
                                     oracle.PEARSON | oracle.F_ABS])
def test_region_max_exhaustive_equals_enumeration(measure):
    spec, f = _c1_field()
    boxes = synth.bricks_of(synth.C1)
    A, B = synth.context_pairs(boxes)
    mx, arg = oracle.region_max(f, None, (8, 8, 4), measure, 3, A, B, 0, 0)
    for r in range(len(A)):
        pa = [((z * 8 + y) * 8 + x) for z in range(A[r][2], A[r][5]) for y in range(A[r][1], A[r][4])
              for x in range(A[r][0], A[r][3])]
        pb = [((z * 8 + y) * 8 + x) for z in range(B[r][2], B[r][5]) for y in range(B[r][1], B[r][4])
              for x in range(B[r][0], B[r][3])]
        ia = np.repeat(pa, len(pb))
        ib = np.tile(pb, len(pa))
        v = oracle.eval_pairs(f, None, measure, 3, ia, ib).astype(np.float32).astype(np.float64)
        if measure & oracle.F_ABS:
            v = np.abs(v)
        v = np.where(np.isnan(v), -np.inf, v)
        q = int(np.argmax(v))  # first maximum = lowest q
        assert mx[r] == v[q]
        assert tuple(arg[r]) == (ia[q], ib[q])


def test_region_max_sampled_matches_sample_list():
    spec, f = _c1_field()
    boxes = synth.bricks_of(synth.C1)
    A, B = synth.context_pairs(boxes)
    S = 50
    mx, arg = oracle.region_max(f, None, (8, 8, 4), oracle.KSG, 3, A, B, S, 99)
    for r in range(len(A)):
        ab = [oracle.sample(99, A[r], B[r], s, 8, 8) for s in range(S)]
        v = oracle.eval_pairs(f, None, oracle.KSG, 3, [a for a, _ in ab], [b for _, b in ab])
        v = v.astype(np.float32).astype(np.float64)
        v = np.where(np.isnan(v), -np.inf, v)
        q = int(np.argmax(v))
        assert mx[r] == v[q] and tuple(arg[r]) == ab[q]
    # a shard (sub-list) of the region pairs gives identical results
    mx2, arg2 = oracle.region_max(f, None, (8, 8, 4), oracle.KSG, 3, A[2:5], B[2:5], S, 99)
    assert np.array_equal(mx2, mx[2:5]) and np.array_equal(arg2, arg[2:5])


def test_region_max_self_pairs_excluded_and_all_nan():
    spec, f = _c1_field()
    box = (0, 0, 0, 2, 1, 1)
    mx, arg = oracle.region_max(f, None, (8, 8, 4), oracle.PEARSON, 3, [box], [box], 0, 0)
    assert tuple(arg[0]) == (0, 1) or tuple(arg[0]) == (1, 0)
    g = f.copy()
    g[:, 0] = 1.0  # constant series -> NaN
    one = (0, 0, 0, 1, 1, 1)
    mx, arg = oracle.region_max(g, None, (8, 8, 4), oracle.PEARSON, 3, [one], [(1, 0, 0, 2, 1, 1)], 0, 0)
    assert np.isnan(mx[0]) and tuple(arg[0]) == (-1, -1)


def test_cluster_centres_pearson_max_is_one():
    spec, f = _c1_field()
    c0, c1 = spec.clusters[0], spec.clusters[3]
    A = (c0.x, c0.y, c0.z, c0.x + 1, c0.y + 1, c0.z + 1)
    B = (c1.x - 1, c1.y - 1, c1.z, c1.x + 1, c1.y + 1, c1.z + 1)
    mx, arg = oracle.region_max(f, None, (8, 8, 4), oracle.PEARSON, 3, [A], [B], 0, 0)
    assert abs(mx[0] - 1.0) < 1e-6
    pb = (c1.z * 8 + c1.y) * 8 + c1.x
    assert arg[0][1] == pb


@pytest.mark.parametrize("absval", [False, True])
def test_pearson_block_max_matmul_equals_brute_force(absval):
    """The oracle's library-matmul block max (used at full brick size) against the plain C
    brute force over every pair (two independent implementations of PAPER.md:133/169)."""
    spec, f = _c1_field()
    boxes = synth.bricks_of(synth.C1)
    A, B = synth.context_pairs(boxes)
    A.append((0, 0, 0, 8, 8, 2))
    B.append((0, 0, 0, 8, 8, 2))  # overlapping boxes: self pairs skipped
    measure = oracle.PEARSON | (oracle.F_ABS if absval else 0)
    mx, arg = oracle.region_max(f, None, (8, 8, 4), measure, 0, A, B, 0, 0)
    for r in range(len(A)):
        v, ab = oracle.pearson_block_max(f, None, (8, 8, 4), A[r], B[r], absval=absval, chunk=7)
        assert abs(v - mx[r]) <= 1e-7
        if v == mx[r]:
            assert ab == tuple(arg[r])
    spec2 = synth.spec_of(synth.C1, 2)
    g = synth.generate(spec2).numpy()
    A2, B2 = synth.matrix_pairs(boxes)
    mx, arg = oracle.region_max(f, g, (8, 8, 4), oracle.PEARSON, 0, A2, B2, 0, 0)
    for r in range(len(A2)):
        v, ab = oracle.pearson_block_max(f, g, (8, 8, 4), A2[r], B2[r])
        assert abs(v - mx[r]) <= 1e-7


@pytest.mark.parametrize("measure,samples", [(oracle.KSG, 0), (oracle.KSG, 40), (oracle.PEARSON, 0),
                                             (oracle.PEARSON | oracle.F_ABS, 25),
                                             (oracle.KSG | oracle.F_KSG_PLUS1, 0)])
def test_region_values_select_max_equals_region_max(measure, samples):
    """The enumeration behind the argmax-margin checks (region_values + select_max) gives the C
    region_max's maximum and argmax exactly; the runner-up is the best value of any OTHER point
    pair, checked by brute force over the enumerated list (ties: margin 0)."""
    spec, f = _c1_field()
    A, B = synth.context_pairs(synth.bricks_of(synth.C1))
    mx, arg = oracle.region_max(f, None, (8, 8, 4), measure, 3, A, B, samples, 5)
    vals, va, vb = oracle.region_values(f, None, (8, 8, 4), measure, 3, A, B, samples, 5)
    smx, sarg, second = oracle.select_max(vals, va, vb)
    assert np.array_equal(smx, mx, equal_nan=True) and np.array_equal(sarg, arg)
    for r in range(len(A)):
        v = np.where(np.isnan(vals[r]), -np.inf, vals[r])
        others = [v[t] for t in range(v.size) if (va[r][t], vb[r][t]) != tuple(arg[r])]
        assert second[r] == (max(others) if others else -np.inf)
        assert second[r] <= smx[r]
        if samples:
            ab = [oracle.sample(5, A[r], B[r], s, 8, 8) for s in range(samples)]
            assert ab == list(zip(va[r].tolist(), vb[r].tolist()))


def test_sample_many_equals_sample():
    A, B = synth.context_pairs(synth.bricks_of(synth.C3))
    A, B = A[::97], B[::97]
    a, b = oracle.sample_many(11, A, B, 30, 250, 352, s0=7)
    for r in range(len(A)):
        for s in range(30):
            assert oracle.sample(11, A[r], B[r], 7 + s, 250, 352) == (a[r, s], b[r, s])


def test_pearson_block_runner_up_brute_force():
    spec, f = _c1_field()
    boxes = synth.bricks_of(synth.C1)
    A, B = synth.context_pairs(boxes)
    vals, va, vb = oracle.region_values(f, None, (8, 8, 4), oracle.PEARSON, 0, A, B, 0, 0)
    _, _, second = oracle.select_max(vals, va, vb)
    for r in range(len(A)):
        v, ab, sec = oracle.pearson_block_max(f, None, (8, 8, 4), A[r], B[r], chunk=5, runner_up=True)
        assert abs(sec - second[r]) <= 1e-7 and sec <= v
