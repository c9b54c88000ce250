"""Pins for the oracle's mean-tree level (§3.3)."""
import numpy as np

import oracle
from conftest import read_golden
from paper_2309_03308_b200 import synth


def test_spec_example():
    row = read_golden("meantree_spec_example.txt")[0]
    vals = np.array([[float(v) for v in row[0].split()]], np.float32)  # one member, 2x2x2
    assert oracle.aggregate_mean(vals, (2, 2, 2), 2, 2, 2)[0, 0] == float(row[1])


def test_constant_field_and_boundary_blocks():
    v = np.full((3, 5 * 3 * 2), 7.25, np.float32)
    g = oracle.aggregate_mean(v, (5, 3, 2), 2, 2, 2)  # ragged: 3 x 2 x 1 coarse points
    assert g.shape == (3, 6) and (g == 7.25).all()
    x = np.arange(5, dtype=np.float32)[None, :]
    g = oracle.aggregate_mean(x, (5, 1, 1), 2, 1, 1)
    assert g.tolist() == [[0.5, 2.5, 4.0]]  # the last block has one point


def test_telescoping():
    spec = synth.field_spec(16, 8, 8, 5, seed=3)
    v = synth.generate(spec).numpy()
    g2 = oracle.aggregate_mean(v, (16, 8, 8), 2, 2, 2)
    g4 = oracle.aggregate_mean(v, (16, 8, 8), 4, 4, 4)
    g22 = oracle.aggregate_mean(g2, (8, 4, 4), 2, 2, 2)
    assert np.max(np.abs(g4 - g22) / np.abs(g4)) < 1e-6
