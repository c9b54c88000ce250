"""CPU checks of the argmax-margin rule used by the GPU parity tests (tests/parity_helpers.py)."""
import numpy as np
import pytest

from parity_helpers import assert_region_argmax, enumerated_value_at


def _value_at(table):
    return lambda r, ab: table.get((r, ab))


def test_margin_rule():
    ref_max, ref_arg = np.array([1.0, 0.5, np.nan]), np.array([[1, 2], [3, 4], [-1, -1]])
    second = np.array([0.9, 0.49999, -np.inf])
    # exact argmax required in region 0 (margin 0.1 > tol), free in region 1 (margin 1e-5 <= tol)
    assert_region_argmax([1.0, 0.5, np.nan], [[1, 2], [5, 6], [-1, -1]], ref_max, ref_arg, second, 1e-4,
                         _value_at({(1, (5, 6)): 0.49999}))
    with pytest.raises(AssertionError):
        assert_region_argmax([1.0, 0.5, np.nan], [[1, 3], [3, 4], [-1, -1]], ref_max, ref_arg, second, 1e-4,
                             _value_at({(0, (1, 3)): 0.99995}))
    with pytest.raises(AssertionError):  # a pair that is not a candidate of the region
        assert_region_argmax([1.0, 0.5, np.nan], [[1, 2], [7, 7], [-1, -1]], ref_max, ref_arg, second, 1e-4,
                             _value_at({}))
    with pytest.raises(AssertionError):  # max off by more than tol
        assert_region_argmax([1.0002, 0.5, np.nan], [[1, 2], [3, 4], [-1, -1]], ref_max, ref_arg, second, 1e-4,
                             _value_at({}))
    with pytest.raises(AssertionError):  # all-NaN region must report (-1, -1)
        assert_region_argmax([1.0, 0.5, np.nan], [[1, 2], [3, 4], [0, 0]], ref_max, ref_arg, second, 1e-4,
                             _value_at({}))


def test_enumerated_value_at():
    vals = [np.array([0.1, np.nan, 0.3])]
    f = enumerated_value_at(vals, [np.array([1, 2, 3])], [np.array([4, 5, 6])])
    assert f(0, (3, 6)) == 0.3 and f(0, (2, 5)) is None and f(0, (9, 9)) is None
