"""Scan protocols (the reference's src/scan.cpp / scan.hpp) through the C ABI
(odegpu_scan_run, implemented by include/odegpu/scan.hpp on the device
pipeline). Same spec fields, defaults, columns, rows and diagnostics as the
reference; this module only marshals."""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import abi
from .api import check

LINEAR, LOG = "linear", "log"


@dataclass
class ParamRange:  # scan.hpp:18-26
    min: float = 0.0
    max: float = 0.0
    res: int = 1
    scale: str = LINEAR

    def to_c(self):
        return abi.ParamRangeC(self.min, self.max, self.res, 1 if self.scale == LOG else 0, 0)

    def values(self) -> np.ndarray:
        out = np.zeros(max(self.res, 1))
        check(abi.load().odegpu_param_range_values(C.byref(self.to_c()), abi.dptr(out)))
        return out


@dataclass
class SolveOptions:  # scan.hpp:29-38
    algorithm: int = abi.RKCK45
    dt: float = 1e-3
    rel_tol: float = 1e-9
    abs_tol: float = 1e-9
    event_tol: float = 1e-6
    batch_capacity: int = 0
    device: int = 0
    devices: tuple = ()  # more than one: whole chunks spread over these devices

    def to_c(self):
        # the device list lives on this object: the C struct is copied by value
        self._devs = (C.c_int32 * max(len(self.devices), 1))(*self.devices)
        return abi.ScanOptions(self.algorithm, self.device, self.dt, self.rel_tol, self.abs_tol, self.event_tol,
                               self.batch_capacity,
                               C.cast(self._devs, C.POINTER(C.c_int32)) if self.devices else None,
                               len(self.devices), 0)


@dataclass
class DuffingScanSpec:  # scan.hpp:59-69
    k: ParamRange = field(default_factory=lambda: ParamRange(0.2, 0.3, 256))
    forcing_amplitude: float = 0.3
    stiffness: float = 1.0
    forcing_omega: float = 1.0
    ic: tuple = (0.0, 0.0)
    transient: int = 1024
    saved: int = 32
    solver: SolveOptions = field(default_factory=SolveOptions)

    def to_c(self):
        return abi.DuffingScanC(self.k.to_c(), self.forcing_amplitude, self.stiffness, self.forcing_omega,
                                (C.c_double * 2)(*self.ic), self.transient, self.saved, self.solver.to_c())


@dataclass
class BubbleScanSpec:  # scan.hpp:73-87 (material: water, a 10 micron bubble)
    pa1_bar: ParamRange = field(default_factory=lambda: ParamRange(1.1, 1.1, 1))
    pa2_bar: ParamRange = field(default_factory=lambda: ParamRange(0.7, 0.7, 1))
    f1_khz: ParamRange = field(default_factory=lambda: ParamRange(20.0, 1000.0, 32, LOG))
    f2_khz: ParamRange = field(default_factory=lambda: ParamRange(20.0, 1000.0, 32, LOG))
    material: dict = field(default_factory=lambda: dict(R_E=10e-6, c_L=1497.3, rho_L=997.1, P_inf=1.0e5,
                                                        p_V=3166.8, sigma=0.072, mu_L=8.902e-4, gamma=1.4,
                                                        theta=0.0))
    ic: tuple = (1.0, 0.0)
    t_end: float = 1e6
    transient: int = 64
    saved: int = 8
    solver: SolveOptions = field(default_factory=lambda: SolveOptions(rel_tol=1e-10, abs_tol=1e-10))

    def to_c(self):
        m = self.material
        return abi.BubbleScanC(self.pa1_bar.to_c(), self.pa2_bar.to_c(), self.f1_khz.to_c(), self.f2_khz.to_c(),
                               m["R_E"], m["c_L"], m["rho_L"], m["P_inf"], m["p_V"], m["sigma"], m["mu_L"],
                               m["gamma"], m["theta"], (C.c_double * 2)(*self.ic), self.t_end, self.transient,
                               self.saved, self.solver.to_c())


@dataclass
class ValveScanSpec:  # scan.hpp:89-105
    q: ParamRange = field(default_factory=lambda: ParamRange(0.2, 10.0, 256))
    kappa: float = 1.25
    delta: float = 10.0
    beta: float = 20.0
    restitution: float = 0.8
    ic: tuple = (0.2, 0.0, math.nan)
    t_end: float = 1e6
    transient: int = 256
    saved: int = 32
    solver: SolveOptions = field(default_factory=lambda: SolveOptions(rel_tol=1e-10, abs_tol=1e-10))

    def to_c(self):
        return abi.ValveScanC(self.q.to_c(), self.kappa, self.delta, self.beta, self.restitution,
                              (C.c_double * 3)(*self.ic), self.t_end, self.transient, self.saved, self.solver.to_c())


@dataclass
class ScanResult:  # scan.hpp:53-57
    columns: list
    rows: np.ndarray
    diagnostics: dict


COLUMNS = {
    abi.SCAN_DUFFING_POINCARE: ["k", "B", "y1", "y2", "status"],
    abi.SCAN_DUFFING_MAXIMA_ACCESSORY: ["k", "y1_max", "status"],
    abi.SCAN_DUFFING_MAXIMA_EVENT: ["k", "y1_max", "status"],
    abi.SCAN_DUFFING_LYAPUNOV: ["k", "lambda_max", "status"],
    abi.SCAN_BUBBLE: ["omega1_radps", "omega2_radps", "pa1_pa", "pa2_pa", "y_exp", "status"],
    abi.SCAN_VALVE: ["q", "y1_max", "y1_min", "status"],
}


def expected_rows(protocol: int, spec) -> int:
    """N x saved for the per-iteration protocols, N for Lyapunov / bubble."""
    if protocol == abi.SCAN_BUBBLE:
        n = spec.pa1_bar.res * spec.pa2_bar.res * spec.f1_khz.res * spec.f2_khz.res
        return n
    n = spec.q.res if protocol == abi.SCAN_VALVE else spec.k.res
    return n if protocol == abi.SCAN_DUFFING_LYAPUNOV else n * spec.saved


def diagnostics_dict(d) -> dict:
    return dict(detections=d.detections, detections_outside_zone=d.detections_outside_zone,
                max_residual_ratio=d.max_residual_ratio, secant_failures=d.secant_failures,
                nonfinite_systems=d.nonfinite_systems, reason_counts=list(d.reason_counts),
                start_times_strictly_increase=bool(d.start_times_strictly_increase))


def run(protocol: int, spec, output: str | None = None) -> ScanResult:
    cols = COLUMNS[protocol]
    rows = np.zeros((expected_rows(protocol, spec), len(cols)))
    nr, nc, d = abi.Index(), abi.Index(), abi.ScanDiagnosticsC()
    c_spec = spec.to_c()
    check(abi.load().odegpu_scan_run(protocol, C.byref(c_spec), abi.dptr(rows), rows.shape[0], C.byref(nr),
                                     C.byref(nc), C.byref(d), output.encode() if output else None))
    assert nc.value == len(cols)
    return ScanResult(cols, rows[: nr.value], diagnostics_dict(d))


def run_duffing_poincare(spec: DuffingScanSpec, output=None):
    return run(abi.SCAN_DUFFING_POINCARE, spec, output)


def run_duffing_maxima(spec: DuffingScanSpec, mode: str = "accessory", output=None):
    return run(abi.SCAN_DUFFING_MAXIMA_EVENT if mode == "event" else abi.SCAN_DUFFING_MAXIMA_ACCESSORY, spec,
               output)


def run_duffing_lyapunov(spec: DuffingScanSpec, output=None):
    return run(abi.SCAN_DUFFING_LYAPUNOV, spec, output)


def run_bubble_scan(spec: BubbleScanSpec, output=None):
    return run(abi.SCAN_BUBBLE, spec, output)


def run_valve_scan(spec: ValveScanSpec, output=None):
    return run(abi.SCAN_VALVE, spec, output)
