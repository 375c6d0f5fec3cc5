"""Known-answer tests of the reference test-suite replayed on the C oracle.

Each case restates an assertion of /root/reference/proj/tests/test_*.cpp
(cited per test) so the restatement is pinned to the reference's own KATs,
not only to its outputs.
"""
import ctypes as C
import math

import numpy as np
import pytest

from oracle import pyoracle
from paper_1810_03931_b200 import abi, models

TWO_PI = 2.0 * math.pi


def lib():
    return pyoracle.load("port")


def step(model, alg, t, h, y, p=()):
    y = np.ascontiguousarray(y, dtype=np.float64)
    p = np.ascontiguousarray(p if len(p) else [0.0], dtype=np.float64)
    out = np.zeros_like(y)
    err = np.zeros_like(y)
    nf = C.c_int()
    assert lib().odo_take_step(C.byref(model.to_c()), alg, t, h, abi.vptr(y), abi.vptr(p), abi.vptr(out),
                               abi.vptr(err), C.byref(nf)) == 0
    return out, err, bool(nf.value)


def rhs(model, t, y, p):
    y = np.ascontiguousarray(y, dtype=np.float64)
    p = np.ascontiguousarray(p, dtype=np.float64)
    dy = np.zeros_like(y)
    lib().odo_rhs(C.byref(model.to_c()), t, abi.vptr(y), abi.vptr(p), abi.vptr(dy))
    return dy


def test_rk4_constant_and_cubic():  # test_steppers.cpp:121-139
    out, err, nf = step(models.ConstantDef(0.0), abi.RK4, 0.0, 0.37, [3.5])
    assert out[0] == 3.5 and err[0] == 0.0 and not nf
    out, _, _ = step(models.CubicTimeDef(), abi.RK4, 0.0, 1.0, [0.0])
    assert out[0] == 0.25


def test_rk4_duffing_against_independent_rk4():  # test_steppers.cpp:141-157
    p = [0.2, 0.3, 1.0, 1.0]
    m = models.DuffingSystem()
    f = lambda t, y: rhs(m, t, y, p)
    y0, h = np.zeros(2), 0.01
    k1 = f(0.0, y0)
    k2 = f(h / 2, y0 + h / 2 * k1)
    k3 = f(h / 2, y0 + h / 2 * k2)
    k4 = f(h, y0 + h * k3)
    expect = y0 + h / 6 * (k1 + 2 * k2 + 2 * k3 + k4)
    out, _, _ = step(m, abi.RK4, 0.0, h, y0, p)
    np.testing.assert_allclose(out, expect, rtol=1e-15, atol=0)


def test_rkck45_trivial_and_exponential():  # test_steppers.cpp:159-196
    out, err, _ = step(models.ConstantDef(0.0), abi.RKCK45, 0.0, 0.5, [2.0])
    assert out[0] == 2.0 and err[0] == 0.0
    out, err, _ = step(models.ConstantDef(1.0), abi.RKCK45, 0.0, 0.5, [1.0])
    assert out[0] == pytest.approx(1.5, rel=1e-15) and abs(err[0]) <= 1e-15
    out, err, _ = step(models.ExponentialDef(), abi.RKCK45, 0.0, 0.1, [1.0])
    assert out[0] == pytest.approx(math.exp(0.1), rel=3e-9)
    assert 1e-12 < err[0] < 1e-6
    # independent Cash-Karp transcription (explicit 4th-order solution)
    c = [0, 0, 1 / 5, 3 / 10, 3 / 5, 1, 7 / 8]
    a = [[], [], [0, 1 / 5], [0, 3 / 40, 9 / 40], [0, 3 / 10, -9 / 10, 6 / 5], [0, -11 / 54, 5 / 2, -70 / 27, 35 / 27],
         [0, 1631 / 55296, 175 / 512, 575 / 13824, 44275 / 110592, 253 / 4096]]
    b5 = [0, 37 / 378, 0, 250 / 621, 125 / 594, 0, 512 / 1771]
    b4 = [0, 2825 / 27648, 0, 18575 / 48384, 13525 / 55296, 277 / 14336, 1 / 4]
    k = [0.0] * 7
    for s in range(1, 7):
        arg = 1.0 + sum(0.1 * a[s][j] * k[j] for j in range(1, s))
        k[s] = arg
    y5 = 1.0 + 0.1 * sum(b5[s] * k[s] for s in range(1, 7))
    y4 = 1.0 + 0.1 * sum(b4[s] * k[s] for s in range(1, 7))
    assert out[0] == pytest.approx(y5, rel=1e-15)
    assert err[0] == pytest.approx(abs(y5 - y4), rel=1e-10)


def test_rkck45_nonfinite_flagged():  # test_steppers.cpp:198-211
    _, _, nf = step(models.BlowUpDef(), abi.RKCK45, 0.0, 0.1, [1.0])
    assert nf


def test_error_ratio_brute_force():  # test_steppers.cpp:213-244
    rng = np.random.default_rng(123)
    f = lib().odo_error_ratio
    for _ in range(200):
        n = 1 + int(rng.integers(0, 6))
        err, yo, yn = rng.random(n) * 1e-6, rng.random(n) * 4 - 2, rng.random(n) * 4 - 2
        rel, ab = rng.random(n) * 1e-6 + 1e-12, rng.random(n) * 1e-6 + 1e-12
        expect = 0.0
        for i in range(n):
            r = err[i] / (ab[i] + rel[i] * max(abs(yo[i]), abs(yn[i])))
            expect = max(expect, r)
        assert f(n, *(abi.vptr(np.ascontiguousarray(v)) for v in (err, yo, yn, rel, ab))) == expect
    z = np.zeros(2)
    rel, ab = np.full(2, 1e-6), np.full(2, 1e-9)
    assert f(2, abi.vptr(z), abi.vptr(z), abi.vptr(z), abi.vptr(rel), abi.vptr(ab)) == 0.0
    e = np.array([1e-9, 0.0])
    assert f(2, abi.vptr(e), abi.vptr(z), abi.vptr(z), abi.vptr(rel), abi.vptr(ab)) == 1.0


def control(ratio, h, nonfinite=False, **kw):  # steppers.hpp:176-198
    oc = models.OdeControls.uniform(1, 1e-9, 1e-9)
    for k, v in kw.items():
        setattr(oc, k, v)
    nxt, fatal = C.c_double(), C.c_int()
    acc = lib().odo_control_step(ratio, h, C.byref(oc.to_c()), int(nonfinite), C.byref(nxt), C.byref(fatal))
    return bool(acc), nxt.value, bool(fatal.value)


def test_control_step_limits():  # test_steppers.cpp:246-287
    acc, nxt, _ = control(0.0, 0.01)
    assert acc and nxt == pytest.approx(0.05, rel=1e-15)
    acc, nxt, fatal = control(0.0, 0.01, nonfinite=True)
    assert not acc and not fatal and nxt == pytest.approx(0.001, rel=1e-15)
    acc, nxt, _ = control(1.0, 0.01)
    assert acc and nxt == pytest.approx(0.009, rel=1e-15)
    assert control(0.0, 0.01, max_step=0.02)[1] == 0.02
    assert control(1e12, 0.0091, max_step=0.02, min_step=0.009)[1] == 0.009
    acc, nxt, fatal = control(100.0, 1e-12)
    assert acc and nxt == 1e-12 and not fatal
    assert control(0.0, 1e-12, nonfinite=True)[2]


def secant(model, t, y, p, h, ev, f0, f1, tol, y_best):
    y = np.ascontiguousarray(y, dtype=np.float64)
    p = np.ascontiguousarray(p if len(p) else [0.0], dtype=np.float64)
    yb = np.ascontiguousarray(y_best, dtype=np.float64)
    th, val, conv = C.c_double(), C.c_double(), C.c_int()
    it = lib().odo_locate_secant(C.byref(model.to_c()), abi.RKCK45, t, abi.vptr(y), abi.vptr(p), h, ev, f0, f1, tol,
                                 abi.vptr(yb), C.byref(th), C.byref(val), C.byref(conv))
    return it, th.value, val.value, bool(conv.value), yb


def test_secant_exact_on_linear_event():  # test_events.cpp:113-132
    it, th, val, conv, yb = secant(models.RampDef(1.0, 0.35), 0.0, [0.0], [], 1.0, 0, -0.35, 0.65, 1e-9, [1.0])
    assert conv and it == 1
    assert th == pytest.approx(0.35, rel=1e-12) and abs(val) <= 1e-9 and yb[0] == pytest.approx(0.35, rel=1e-12)


def test_secant_matches_bisection_on_seat_contact():  # test_events.cpp:134-182
    m = models.SeatContactDef()
    p = [1.25, 10.0, 20.0, 0.3, 0.8]
    y0 = [0.5, -2.0, 10.0]
    h = 0.4
    end, _, _ = step(m, abi.RKCK45, 0.0, h, y0, p)
    assert end[0] < 0
    it, th, val, conv, _ = secant(m, 0.0, y0, p, h, 0, y0[0], end[0], 1e-9, end)
    assert conv and abs(val) <= 1e-9
    lo, hi = 0.0, h
    while hi - lo > 1e-12:
        mid = 0.5 * (lo + hi)
        if step(m, abi.RKCK45, 0.0, mid, y0, p)[0][0] > 0:
            lo = mid
        else:
            hi = mid
    assert abs(th - 0.5 * (lo + hi)) <= 1e-9


def test_duffing_rhs_known_values():  # test_models.cpp:81-111
    m = models.DuffingSystem()
    p = [0.2, 0.3, 1.0, 1.0]
    dy = rhs(m, 0.0, [0.0, 0.0], p)
    assert dy[0] == 0.0 and dy[1] == 0.3
    dy = rhs(m, math.pi / 2, [1.0, 0.0], p)
    assert dy[0] == 0.0 and abs(dy[1]) <= 1e-15


def test_keller_miksis_equilibrium_and_breakdown():  # test_models.cpp:212-264 (equilibrium identity)
    from paper_1810_03931_b200.workloads import bubble_coefficients

    c = bubble_coefficients([0.0], [0.0], [TWO_PI * 20e3], [TWO_PI * 20e3])[:, 0]
    dy = rhs(models.KellerMiksisSystem(), 0.0, [1.0, 0.0], c)
    assert dy[0] == 0.0 and abs(dy[1]) <= 1e-9 * abs(c[0])
    dy = rhs(models.KellerMiksisSystem(), 0.0, [-1.0, 0.0], c)
    assert np.isnan(dy).all()


@pytest.mark.parametrize("case,expect", [
    ("unit_slope_rk4", dict(reason=0, accepted=4, final_t=1.0, y0=1.0)),  # test_driver.cpp:48-59
    ("unit_slope_empty", dict(reason=0, accepted=0, final_t=2.5, y0=7.0)),  # :84-94
])
def test_driver_kats(case, expect):
    import golden_io

    g = golden_io.load(f"fake_{case}")
    td, y, p, acc = (g[f"in_{k}"].copy() for k in ("td", "y", "p", "acc"))
    oc, _, _ = pyoracle.solve("port", g["model"], td, y, p, acc, algorithm=int(g["algorithm"]), dt=float(g["dt"]))
    assert oc["reason"][0] == expect["reason"] and oc["accepted_steps"][0] == expect["accepted"]
    assert oc["final_t"][0] == expect["final_t"]
    assert y[0] == pytest.approx(expect["y0"], rel=1e-15)
