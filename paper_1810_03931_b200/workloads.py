"""Synthetic parameter-sweep workloads of SURVEY.md §8(d) (cfg1..cfg5).

Grids follow ParamRange::values (reference src/scan.cpp:17-37): end points
exact, linear points ``min + i*(max-min)/(res-1)``, log points
``min*exp(i*log(max/min)/(res-1))`` evaluated with libm (``math``) so the
values are bitwise those of the reference. The bubble coefficients follow
bubble_coefficients (models/keller_miksis.hpp:47-77) operation by operation.
All data are deterministic; no RNG.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import abi
from .models import (
    BubbleCollapseSystem,
    DuffingMaxEventSystem,
    DuffingMaxMinSystem,
    OdeControls,
    SystemDef,
    ValveSystem,
)

TWO_PI = 2.0 * math.pi


def param_range(lo: float, hi: float, res: int, log: bool = False) -> np.ndarray:
    """ParamRange::values (src/scan.cpp:17-37)."""
    if res < 1:
        raise ValueError("ParamRange: res must be >= 1")
    if res == 1:
        return np.array([lo])
    if log and (not lo > 0 or not hi > 0):
        raise ValueError("ParamRange: log scale requires positive bounds")
    out = np.empty(res)
    for i in range(res):
        if i == 0:
            out[i] = lo
        elif i == res - 1:
            out[i] = hi
        elif not log:
            out[i] = lo + float(i) * (hi - lo) / float(res - 1)
        else:
            out[i] = lo * math.exp(float(i) * math.log(hi / lo) / float(res - 1))
    return out


# BubblePhysical defaults (models/keller_miksis.hpp:18-32), declaration order.
BUBBLE_FIELDS = ("pa1", "pa2", "omega1", "omega2", "theta", "R_E", "c_L", "rho_L", "P_inf", "p_V", "sigma", "mu_L", "gamma")
WATER = dict(pa1=0.0, pa2=0.0, omega1=0.0, omega2=0.0, theta=0.0, R_E=10e-6, c_L=1497.3, rho_L=997.1,
             P_inf=1.0e5, p_V=3166.8, sigma=0.072, mu_L=8.902e-4, gamma=1.4)


def bubble_coefficients(pa1, pa2, omega1, omega2, theta=0.0, **material) -> np.ndarray:
    """Vectorised bubble_coefficients (keller_miksis.hpp:47-77) -> [13, N] (SoA)."""
    phys = dict(WATER)
    phys.update(material)
    pa1, pa2, omega1, omega2 = (np.asarray(v, dtype=np.float64) for v in (pa1, pa2, omega1, omega2))
    theta = np.broadcast_to(np.asarray(theta, dtype=np.float64), omega1.shape)
    if not np.all(omega1 > 0):
        raise ValueError("bubble_coefficients: omega1 must be > 0")
    R_E, c_L, rho_L = phys["R_E"], phys["c_L"], phys["rho_L"]
    P_inf, p_V, sigma, mu_L, gamma = phys["P_inf"], phys["p_V"], phys["sigma"], phys["mu_L"], phys["gamma"]
    w = R_E * omega1
    S = TWO_PI / w
    G = S * S / rho_L
    A = P_inf - p_V
    B = 2.0 * sigma / R_E
    c = np.empty((13,) + omega1.shape)
    c[0] = (A + B) * G
    c[1] = (1.0 - 3.0 * gamma) * (A + B) * S / (rho_L * c_L)
    c[2] = A * G
    c[3] = B * G
    c[4] = 4.0 * mu_L / (rho_L * R_E * R_E) * (TWO_PI / omega1)
    c[5] = pa1 * G
    c[6] = pa2 * G
    c[7] = (w / c_L) * c[5]
    c[8] = (w / c_L) * c[6]
    c[9] = w / (TWO_PI * c_L)
    c[10] = 3.0 * gamma
    c[11] = omega2 / omega1
    c[12] = theta
    return c


@dataclass
class Workload:
    """One synthetic pool plus the solver settings it is run with."""

    name: str
    description: str
    model: SystemDef
    algorithm: int
    dt: float
    iterations: int
    td: np.ndarray  # [2, N]
    y: np.ndarray  # [n, N]
    p: np.ndarray  # [np, N]
    acc: np.ndarray  # [na, N]
    # FP64-pipe instructions per trial step: SURVEY.md §8d's count from the
    # reference formulas, with the controller's pow(ratio, -0.2) (80) costed
    # as the kernels' 13-instruction Newton fifth root
    instr_per_step: int
    flops_per_step: int

    @property
    def n(self) -> int:
        return self.td.shape[1]

    def config(self) -> abi.SolverConfig:
        return abi.SolverConfig(self.algorithm, 0, self.dt, 64, 1)

    def subset(self, idx) -> "Workload":
        """Systems `idx` (slice or index array) as a new, contiguous pool."""
        cp = lambda a: np.ascontiguousarray(a[:, idx])
        return Workload(self.name, self.description, self.model, self.algorithm, self.dt, self.iterations,
                        cp(self.td), cp(self.y), cp(self.p), cp(self.acc), self.instr_per_step, self.flops_per_step)

    def strided(self, count: int) -> "Workload":
        """`count` systems spread evenly over the whole grid (bounded samples)."""
        if count >= self.n:
            return self.subset(slice(None))
        idx = np.unique(np.linspace(0, self.n - 1, count).round().astype(np.int64))
        return self.subset(idx)

    def arrays(self):
        """Flat SoA copies (td, y, p, acc), ready for the C ABI."""
        return tuple(np.ascontiguousarray(a).reshape(-1).copy() for a in (self.td, self.y, self.p, self.acc))


def _grid2(a: np.ndarray, b: np.ndarray):
    """Outer product grid, `a` slow (outer) and `b` fast (inner), like the
    nested loops of run_bubble_scan (src/scan.cpp:253-258)."""
    return np.repeat(a, b.size), np.tile(b, a.size)


def cfg1(n: int = 46_080) -> Workload:
    """Duffing RK4 dt=1e-2, forcing-amplitude sweep, per-period max/min."""
    B = param_range(0.1, 0.5, n)
    p = np.stack([np.full(n, 0.2), B, np.ones(n), np.ones(n)])
    td = np.stack([np.zeros(n), np.full(n, TWO_PI)])
    return Workload("cfg1_duffing_rk4", f"Duffing RK4 dt=1e-2, B sweep, N={n}, 1024 periods, max/min accessories",
                    DuffingMaxMinSystem(), abi.RK4, 1e-2, 1024, td, np.zeros((2, n)), p, np.zeros((4, n)), 105, 181)


def cfg2(nk: int = 1024, nb: int = 1024) -> Workload:
    """Duffing RKCK45 + event F=y2 (local maxima), k x B sweep of 2^20."""
    k, B = _grid2(param_range(0.2, 0.3, nk), param_range(0.1, 0.5, nb))
    n = k.size
    p = np.stack([k, B, np.ones(n), np.ones(n)])
    td = np.stack([np.zeros(n), np.full(n, TWO_PI)])
    model = DuffingMaxEventSystem(1e-6, 0, OdeControls.uniform(2, 1e-9, 1e-9))
    return Workload("cfg2_duffing_rkck45_event", f"Duffing RKCK45 tol 1e-9 + event F=y2, k x B = {nk}x{nb}",
                    model, abi.RKCK45, 1e-3, 32, td, np.zeros((2, n)), p, np.zeros((2, n)), 222, 382)


def cfg3(npa: int = 1024, nf: int = 1024, transient: int = 64, saved: int = 8) -> Workload:
    """Keller-Miksis collapse, PA1 x f1 sweep of 2^20 (scan.hpp:73-87)."""
    pa1_bar, f1_khz = _grid2(param_range(0.5, 1.1, npa), param_range(20.0, 1000.0, nf, log=True))
    w1 = f1_khz * 1e3 * TWO_PI
    c = bubble_coefficients(pa1_bar * 1e5, np.zeros_like(w1), w1, w1)
    n = w1.size
    td = np.stack([np.zeros(n), np.full(n, 1e6)])
    y = np.stack([np.ones(n), np.zeros(n)])
    model = BubbleCollapseSystem(1e-6, OdeControls.uniform(2, 1e-10, 1e-10))
    return Workload("cfg3_keller_miksis", f"Keller-Miksis RKCK45 tol 1e-10 collapse, PA1 x f1 = {npa}x{nf}",
                    model, abi.RKCK45, 1e-3, transient + saved, td, y, c, np.zeros((4, n)), 1194, 1972)


def cfg4(n: int = 1 << 19, transient: int = 256, saved: int = 32) -> Workload:
    """Pressure relief valve with impacts, q sweep of 2^19 (scan.hpp:89-105)."""
    q = param_range(0.2, 10.0, n)
    kappa, delta, beta, r = 1.25, 10.0, 20.0, 0.8
    p = np.stack([np.full(n, kappa), np.full(n, delta), np.full(n, beta), q, np.full(n, r)])
    td = np.stack([np.zeros(n), np.full(n, 1e6)])
    y = np.stack([np.full(n, 0.2), np.zeros(n), np.full(n, delta + 0.2)])
    model = ValveSystem(1e-6, OdeControls.uniform(3, 1e-10, 1e-10))
    return Workload("cfg4_valve", f"Valve RKCK45 tol 1e-10, 2 events + impact action, q sweep N={n}",
                    model, abi.RKCK45, 1e-3, transient + saved, td, y, p, np.zeros((2, n)), 220, 371)


def cfg5(log2n: int) -> Workload:
    """Keller-Miksis scaling sweep: 2^ceil(k/2) PA1 x 2^floor(k/2) f1."""
    return cfg3(1 << ((log2n + 1) // 2), 1 << (log2n // 2))


CONFIGS = {"cfg1": cfg1, "cfg2": cfg2, "cfg3": cfg3, "cfg4": cfg4}
