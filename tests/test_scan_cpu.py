"""Scan-layer host logic without a GPU: ParamRange grids (src/scan.cpp:17-37)
through the product's C ABI against the compiled reference, and the
reference's own scan known answers (tests/test_scan.cpp) on the oracle."""
import math

import numpy as np
import pytest

from oracle import pyoracle
from paper_1810_03931_b200 import abi, scan
from paper_1810_03931_b200.api import InvalidArgument


def ref_values(lo, hi, res, log):
    out = np.zeros(max(res, 1))
    lib = pyoracle.load("reference")
    f = lib.odref_param_range
    import ctypes as C

    f.restype = C.c_int
    f.argtypes = [C.c_double, C.c_double, abi.Index, C.c_int, C.POINTER(C.c_double)]
    assert f(lo, hi, res, int(log), out.ctypes.data_as(C.POINTER(C.c_double))) == 0
    return out


@pytest.mark.parametrize("lo,hi,res,log", [(0.2, 0.3, 256, False), (20.0, 1000.0, 32, True), (1.1, 1.1, 1, False),
                                           (0.5, 1.1, 1024, False), (20.0, 1000.0, 1024, True), (-3.0, 7.0, 2, False)])
def test_param_range_matches_reference_bitwise(lo, hi, res, log):
    mine = scan.ParamRange(lo, hi, res, scan.LOG if log else scan.LINEAR).values()
    assert np.array_equal(mine.view(np.uint64), ref_values(lo, hi, res, log).view(np.uint64))
    assert mine[0] == lo and mine[-1] == (hi if res > 1 else lo)  # end points exact


def test_param_range_errors():  # scan.cpp:18-22
    with pytest.raises(InvalidArgument, match="res must be >= 1"):
        scan.ParamRange(0, 1, 0).values()
    with pytest.raises(InvalidArgument, match="log scale requires positive bounds"):
        scan.ParamRange(0.0, 1.0, 4, scan.LOG).values()


def test_expected_row_counts():
    d = scan.DuffingScanSpec(k=scan.ParamRange(0.2, 0.3, 10), transient=3, saved=4)
    assert scan.expected_rows(abi.SCAN_DUFFING_POINCARE, d) == 40
    assert scan.expected_rows(abi.SCAN_DUFFING_LYAPUNOV, d) == 10
    b = scan.BubbleScanSpec(pa1_bar=scan.ParamRange(1, 2, 3), f1_khz=scan.ParamRange(20, 40, 5, scan.LOG),
                            f2_khz=scan.ParamRange(20, 20, 1))
    assert scan.expected_rows(abi.SCAN_BUBBLE, b) == 15


def test_reference_bubble_scan_known_answer():
    """test_scan.cpp's bubble smoke: every saved-or-transient iteration of every
    system ends in EventStop (reason_counts[EventStop] == systems x iterations)."""
    spec = scan.BubbleScanSpec(pa1_bar=scan.ParamRange(1.1, 1.1, 1), pa2_bar=scan.ParamRange(0.7, 0.7, 1),
                               f1_khz=scan.ParamRange(20, 1000, 3, scan.LOG), f2_khz=scan.ParamRange(20, 1000, 3,
                                                                                                   scan.LOG),
                               transient=4, saved=4)
    rows, d = pyoracle.scan(abi.SCAN_BUBBLE, spec)
    assert rows.shape == (9, 6)
    assert d["reason_counts"][abi.EVENT_STOP] == 9 * 8
    assert d["start_times_strictly_increase"]
    assert np.all(rows[:, 5] == 0)
