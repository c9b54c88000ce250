"""Pins for the oracle's PPMCC and digamma (CPU only).

PPMCC: PAPER.md:169 (§3.2).  Digamma: PAPER.md:174-178 (Eq. 2).
Pins: SPEC worked examples (golden), numpy.corrcoef (library routine), affine
closed form, symmetry; scipy.special.digamma (library routine), Euler-gamma and
recurrence (golden).
"""
import math

import numpy as np
import pytest
import scipy.special

import oracle
from conftest import read_golden


@pytest.mark.parametrize("row", read_golden("ppmcc_spec_examples.txt"))
def test_ppmcc_spec_examples(row):
    x = [float(v) for v in row[0].split()]
    y = [float(v) for v in row[1].split()]
    assert oracle.ppmcc(x, y) == pytest.approx(float(row[2]), abs=1e-15)


def test_ppmcc_matches_numpy_corrcoef():
    rng = np.random.default_rng(11)
    for n in (10, 100, 1000):
        for _ in range(20):
            x = (250 + rng.standard_normal(n)).astype(np.float32)
            y = (0.3 * x + rng.standard_normal(n)).astype(np.float32)
            ref = np.corrcoef(x.astype(np.float64), y.astype(np.float64))[0, 1]
            assert abs(oracle.ppmcc(x, y) - ref) < 1e-12


def test_ppmcc_affine_closed_form_and_symmetry():
    rng = np.random.default_rng(12)
    for n in (10, 100, 1000):
        x = rng.standard_normal(n).astype(np.float32)
        for a, b in ((2.5, 1.0), (-0.75, 3.0)):
            y = (np.float32(a) * x + np.float32(b)).astype(np.float32)
            assert abs(oracle.ppmcc(x, y) - math.copysign(1.0, a)) < 1e-6
        y = rng.standard_normal(n).astype(np.float32)
        assert oracle.ppmcc(x, y) == oracle.ppmcc(y, x)
        assert oracle.ppmcc(x, x) == pytest.approx(1.0, abs=1e-15)


def test_ppmcc_zero_variance_is_nan():
    assert math.isnan(oracle.ppmcc([1, 1, 1, 1], [1, 2, 3, 4]))
    assert math.isnan(oracle.ppmcc([1, 2, 3, 4], [7, 7, 7, 7]))


@pytest.mark.parametrize("row", read_golden("digamma_values.txt"))
def test_digamma_golden(row):
    assert oracle.digamma_int(int(row[0])) == pytest.approx(float(row[1]), abs=1e-14)


def test_digamma_matches_scipy_and_recurrence():
    for m in range(1, 2002):
        assert abs(oracle.digamma_int(m) - scipy.special.digamma(m)) < 1e-12
        assert abs(oracle.digamma_int(m + 1) - oracle.digamma_int(m) - 1.0 / m) < 1e-12
    assert math.isnan(oracle.digamma_int(0))
