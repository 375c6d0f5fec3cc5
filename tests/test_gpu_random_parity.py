"""Randomised parity: seeded random parameters, time domains, initial states,
tolerances and initial steps for every built-in model, GPU against the C
oracle (bitwise-pinned to the reference). Integer outcomes must agree
exactly (they do: 0 mismatches over 20 480 random systems); values as
tests/parity.py's rules, within 1e-6. These inputs are off the
BASELINE grids on purpose — they exercise rejections, clipping, event
location, impacts, equilibria and early stops at arbitrary operating points."""
import math

import numpy as np
import pytest

import parity
from oracle import pyoracle
from paper_1810_03931_b200 import abi, workloads
from paper_1810_03931_b200.models import (BubbleCollapseSystem, DuffingMaxAccessorySystem, DuffingMaxEventSystem,
                                          DuffingMaxMinSystem, OdeControls, ValveSystem)

pytestmark = pytest.mark.gpu

N = 2048


def wl_of(name, model, alg, dt, td, y, p, acc):
    return workloads.Workload(name, name, model, alg, dt, 1, td, y, p, acc, 0, 0)


def duffing_params(rng, n):
    return np.stack([rng.uniform(0.05, 0.5, n), rng.uniform(0.05, 0.6, n), rng.uniform(0.5, 1.5, n),
                     rng.uniform(0.5, 1.5, n)])


def make(case, seed):
    rng = np.random.default_rng(seed)
    n = N
    tol = 10.0 ** rng.uniform(-10, -7)
    ode = lambda dim: OdeControls.uniform(dim, tol, tol)
    if case == "duffing_event":
        t1 = rng.uniform(1.0, 12.0, n)
        td = np.stack([np.zeros(n), t1])
        y = np.stack([rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)])
        return wl_of(case, DuffingMaxEventSystem(10.0 ** rng.uniform(-7, -5), int(rng.integers(0, 3)), ode(2)),
                     abi.RKCK45, 10.0 ** rng.uniform(-4, -1), td, y, duffing_params(rng, n), np.zeros((2, n)))
    if case == "duffing_accessory":
        td = np.stack([rng.uniform(-3, 3, n), np.zeros(n)])
        td[1] = td[0] + rng.uniform(0.5, 8.0, n)
        y = np.stack([rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)])
        return wl_of(case, DuffingMaxAccessorySystem(ode(2)), abi.RKCK45, 10.0 ** rng.uniform(-4, -1), td, y,
                     duffing_params(rng, n), np.zeros((2, n)))
    if case == "duffing_rk4":
        td = np.stack([np.zeros(n), rng.uniform(0.5, 7.0, n)])
        y = np.stack([rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)])
        return wl_of(case, DuffingMaxMinSystem(ode(2)), abi.RK4, rng.uniform(0.003, 0.03), td, y,
                     duffing_params(rng, n), np.zeros((4, n)))
    if case == "valve":
        q = rng.uniform(0.2, 10.0, n)
        p = np.stack([rng.uniform(0.8, 1.6, n), rng.uniform(8, 12, n), rng.uniform(15, 25, n), q,
                      rng.uniform(0.5, 0.95, n)])
        td = np.stack([np.zeros(n), np.full(n, 1e6)])
        y = np.stack([rng.uniform(0.0, 0.5, n), rng.uniform(-0.2, 0.2, n), p[1] + rng.uniform(0.0, 0.5, n)])
        return wl_of(case, ValveSystem(10.0 ** rng.uniform(-7, -5), ode(3)), abi.RKCK45, 1e-3, td, y, p,
                     np.zeros((2, n)))
    if case == "bubble":
        pa1 = rng.uniform(0.3e5, 1.2e5, n)
        w1 = 2 * math.pi * 1e3 * 10.0 ** rng.uniform(math.log10(20), 3, n)
        c = workloads.bubble_coefficients(pa1, rng.uniform(0, 0.5e5, n), w1, w1 * rng.uniform(0.5, 2.0, n))
        td = np.stack([np.zeros(n), np.full(n, 1e6)])
        y = np.stack([np.ones(n), np.zeros(n)])
        return wl_of(case, BubbleCollapseSystem(1e-6, OdeControls.uniform(2, 1e-10, 1e-10)), abi.RKCK45, 1e-3, td,
                     y, c, np.zeros((4, n)))
    raise ValueError(case)


RULES = {
    "duffing_event": dict(time_acc={1: 0}),
    "duffing_accessory": dict(time_acc={1: 0}),
    "duffing_rk4": dict(time_acc={1: 0, 3: 2}),
    "valve": dict(pinned_state=(1,), pinned_acc=(1,)),
    "bubble": dict(pinned_state=(1,), time_acc={0: 1, 2: 3}),
}


@pytest.mark.parametrize("case", sorted(RULES))
@pytest.mark.parametrize("seed", [1, 2])
def test_random_inputs_match_oracle(case, seed):
    wl = make(case, 1000 * seed + len(case))
    got = parity.run_gpu(wl, 1)
    ref = pyoracle.solve_workload("port", wl, 1)
    rep = parity.compare(wl, got, ref, **RULES[case])
    for k in parity.COUNT_FIELDS:
        assert rep[f"mismatch_{k}"] == 0, (k, rep)
    # horizons up to two forcing periods at random (partly chaotic) Duffing
    # parameters, and event-pinned stop states for random stop counts: the
    # value bar is the chaotic short-horizon one
    assert rep["worst_rel"] <= 1e-6, rep
