"""Scan protocols on the device pipeline (include/odegpu/scan.hpp) against
the reference's own src/scan.cpp (oracle/_ref), protocol by protocol.

Rows come in the reference's order (chunk, saved iteration, system). The
parameter columns are bit-identical (same ParamRange / grid arithmetic on the
host); statuses, and the diagnostics' counts (reason counts per iteration,
detections, secant failures, non-finite systems, detections outside the
zone, the start-time check) are exact; value columns within the solver
parity tolerance of tests/test_gpu_parity.py at these horizons (chaotic
Duffing sets over a few periods), max |F|/tol within 1e-6 relative."""
import math

import numpy as np
import pytest

from oracle import pyoracle
from paper_1810_03931_b200 import abi, scan

pytestmark = pytest.mark.gpu


def compare(protocol, spec, param_cols, value_cols, rtol, atol=1e-9):
    got = scan.run(protocol, spec)
    rows, d = pyoracle.scan(protocol, spec)
    assert got.rows.shape == rows.shape
    status = got.rows.shape[1] - 1
    assert np.array_equal(got.rows[:, param_cols].view(np.uint64), rows[:, param_cols].view(np.uint64))
    assert np.array_equal(got.rows[:, status], rows[:, status])
    err = np.abs(got.rows[:, value_cols] - rows[:, value_cols]) / (np.abs(rows[:, value_cols]) + atol)
    assert err.max() <= rtol, f"max rel err {err.max():.3e}"
    g = got.diagnostics
    for k in ("detections", "detections_outside_zone", "secant_failures", "nonfinite_systems", "reason_counts",
              "start_times_strictly_increase"):
        assert g[k] == d[k], (k, g[k], d[k])
    assert g["max_residual_ratio"] == pytest.approx(d["max_residual_ratio"], rel=1e-6, abs=1e-12)
    return got, rows, d


def duffing_spec(cap=0, transient=4, saved=3, res=96):
    return scan.DuffingScanSpec(k=scan.ParamRange(0.2, 0.3, res), transient=transient, saved=saved,
                                solver=scan.SolveOptions(batch_capacity=cap))


@pytest.mark.parametrize("cap", [0, 40])  # one chunk / three chunks of the pool
def test_duffing_poincare(cap):
    compare(abi.SCAN_DUFFING_POINCARE, duffing_spec(cap), [0, 1], [2, 3], 1e-7)


@pytest.mark.parametrize("protocol", [abi.SCAN_DUFFING_MAXIMA_ACCESSORY, abi.SCAN_DUFFING_MAXIMA_EVENT])
def test_duffing_maxima(protocol):
    got, rows, d = compare(protocol, duffing_spec(32), [0], [1], 1e-7)
    if protocol == abi.SCAN_DUFFING_MAXIMA_EVENT:
        assert d["detections"] > 0 and d["detections_outside_zone"] == 0


def test_duffing_lyapunov():
    spec = duffing_spec(0, transient=2, saved=4, res=32)
    compare(abi.SCAN_DUFFING_LYAPUNOV, spec, [0], [1], 1e-6)


def test_bubble_scan():
    spec = scan.BubbleScanSpec(pa1_bar=scan.ParamRange(0.5, 1.1, 4), pa2_bar=scan.ParamRange(0.0, 0.7, 2),
                               f1_khz=scan.ParamRange(20.0, 1000.0, 6, scan.LOG),
                               f2_khz=scan.ParamRange(20.0, 1000.0, 2, scan.LOG), transient=6, saved=4,
                               solver=scan.SolveOptions(rel_tol=1e-10, abs_tol=1e-10, batch_capacity=40))
    got, rows, d = compare(abi.SCAN_BUBBLE, spec, [0, 1, 2, 3], [4], 1e-6)
    assert d["reason_counts"][abi.EVENT_STOP] == rows.shape[0] * 10
    assert d["start_times_strictly_increase"]


def test_valve_scan():
    spec = scan.ValveScanSpec(q=scan.ParamRange(0.2, 10.0, 128), transient=16, saved=6,
                              solver=scan.SolveOptions(rel_tol=1e-10, abs_tol=1e-10, batch_capacity=50))
    compare(abi.SCAN_VALVE, spec, [0], [1, 2], 1e-6, atol=1e-6)


def test_csv_round_trip(tmp_path):
    """emit_rows: '# ' header, %.16e fields — parsing back is lossless
    (test_scan.cpp's round-trip check)."""
    path = tmp_path / "maxima.csv"
    got = scan.run(abi.SCAN_DUFFING_MAXIMA_ACCESSORY, duffing_spec(0, 2, 2, 16), str(path))
    lines = path.read_text().splitlines()
    assert lines[0] == "# k,y1_max,status"
    back = np.array([[float(v) for v in ln.split(",")] for ln in lines[1:]])
    assert np.array_equal(back, got.rows)
    import re

    assert all(re.fullmatch(r"-?\d\.\d{16}e[+-]\d{2,3}", f) for ln in lines[1:] for f in ln.split(","))


@pytest.mark.parametrize("protocol", [abi.SCAN_DUFFING_POINCARE, abi.SCAN_VALVE, abi.SCAN_BUBBLE])
def test_multi_device_scan_equals_single_device(protocol):
    """Whole chunks spread over several devices (here two pipelines on device
    0) give the one-device rows and diagnostics bit for bit."""
    if protocol == abi.SCAN_BUBBLE:
        mk = lambda devs: scan.BubbleScanSpec(pa1_bar=scan.ParamRange(0.5, 1.1, 5), pa2_bar=scan.ParamRange(0, 0, 1),
                                             f1_khz=scan.ParamRange(20, 1000, 7, scan.LOG),
                                             f2_khz=scan.ParamRange(20, 20, 1), transient=3, saved=2,
                                             solver=scan.SolveOptions(rel_tol=1e-10, abs_tol=1e-10,
                                                                      batch_capacity=8, devices=devs))
    elif protocol == abi.SCAN_VALVE:
        mk = lambda devs: scan.ValveScanSpec(q=scan.ParamRange(0.2, 10.0, 70), transient=4, saved=3,
                                            solver=scan.SolveOptions(rel_tol=1e-10, abs_tol=1e-10,
                                                                     batch_capacity=16, devices=devs))
    else:
        mk = lambda devs: scan.DuffingScanSpec(k=scan.ParamRange(0.2, 0.3, 77), transient=3, saved=2,
                                              solver=scan.SolveOptions(batch_capacity=20, devices=devs))
    one = scan.run(protocol, mk(()))
    many = scan.run(protocol, mk((0, 0, 0)))
    assert np.array_equal(one.rows.view(np.uint64), many.rows.view(np.uint64))
    assert one.diagnostics == many.diagnostics
