"""max / mean aggregation definitions (oracle/aggregators.py) on known answers (CPU), and the
host-side mean coefficients of the C ABI against them."""
import ctypes as C

import numpy as np

from aggregators import max_bwd, max_fwd, mean_coefficients, mean_fwd


def _star():
    # rows: 0 <- {1, 2, 3}, 1 <- {0}, 2 <- {} (empty), 3 <- {0, 0} (duplicate edge: tie)
    rowptr = np.array([0, 3, 4, 4, 6], np.int32)
    cols = np.array([1, 2, 3, 0, 0, 0], np.int32)
    x = np.array([[1.0, -2.0], [3.0, 5.0], [3.0, -1.0], [0.5, 5.0]], np.float32)
    return rowptr, cols, x


def test_max_known_answers():
    rowptr, cols, x = _star()
    y, arg = max_fwd(rowptr, cols, x)
    assert np.array_equal(y, np.array([[3.0, 5.0], [1.0, -2.0], [0.0, 0.0], [1.0, -2.0]], np.float32))
    # ties keep the first occurrence (edge 0 in col 0, edge 0 in col 1 for row 0; edge 4 for row 3)
    assert np.array_equal(arg, np.array([[0, 0], [3, 3], [-1, -1], [4, 4]], np.int32))
    gy = np.ones((4, 2), np.float32)
    gx = max_bwd(rowptr, cols, arg, gy, 4)
    # source 0 is the argmax of rows 1 and 3 (both columns); source 1 of row 0
    assert np.array_equal(gx, np.array([[2.0, 2.0], [1.0, 1.0], [0.0, 0.0], [0.0, 0.0]], np.float32))


def test_mean_known_answers_and_abi_coefficients():
    from paper_2106_05609_b200._native import check, lib
    rowptr, cols, x = _star()
    y = mean_fwd(rowptr, cols, x)
    assert np.allclose(y[0], (x[1] + x[2] + x[3]) / 3) and np.array_equal(y[2], [0.0, 0.0])
    assert np.array_equal(y[3], x[0])
    cf = np.zeros(len(cols), np.float32)
    check(lib.gasb_mean_coefficients(rowptr.ctypes.data, len(rowptr) - 1, cf.ctypes.data))
    assert np.array_equal(cf, mean_coefficients(rowptr))
    assert cf[0] == np.float32(1.0 / 3.0) and cf[4] == np.float32(0.5)
