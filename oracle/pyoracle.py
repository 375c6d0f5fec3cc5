"""ctypes loaders for the two CPU checkers — TEST INFRASTRUCTURE ONLY.

* ``port``      : oracle/_build/libodeoracle.so, the plain-C restatement
                  (oracle/odeoracle.c), single-threaded.
* ``reference`` : oracle/_ref/libodref.so, the unmodified reference solver
                  compiled from /root/reference/proj by oracle/Makefile.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this module.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

from paper_1810_03931_b200 import abi

HERE = Path(__file__).resolve().parent
PORT_LIB = HERE / "_build" / "libodeoracle.so"
REF_LIB = HERE / "_ref" / "libodref.so"

_libs: dict[str, C.CDLL] = {}

_SOLVE_ARGS = [
    C.POINTER(abi.Model), abi.Index, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int,
    C.POINTER(abi.SolverConfig), C.POINTER(abi.OdeControls), abi.Index, C.c_void_p, C.c_void_p, C.c_void_p,
    C.c_void_p, C.POINTER(C.c_double),
]


def available(which: str) -> bool:
    return (PORT_LIB if which == "port" else REF_LIB).exists()


def load(which: str) -> C.CDLL:
    if which not in _libs:
        path = PORT_LIB if which == "port" else REF_LIB
        if not path.exists():
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        lib = C.CDLL(str(path))
        prefix = "odo" if which == "port" else "odref"
        f = getattr(lib, f"{prefix}_solve")
        f.restype = C.c_int
        f.argtypes = _SOLVE_ARGS
        e = getattr(lib, f"{prefix}_last_error")
        e.restype = C.c_char_p
        bc = getattr(lib, f"{prefix}_bubble_coefficients")
        bc.restype = C.c_int
        bc.argtypes = [abi.Index, C.c_void_p, C.c_void_p]
        if which == "port":
            lib.odo_take_step.restype = C.c_int
            lib.odo_take_step.argtypes = [C.POINTER(abi.Model), C.c_int, C.c_double, C.c_double, C.c_void_p,
                                          C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_int)]
            lib.odo_error_ratio.restype = C.c_double
            lib.odo_error_ratio.argtypes = [C.c_int] + [C.c_void_p] * 5
            lib.odo_control_step.restype = C.c_int
            lib.odo_control_step.argtypes = [C.c_double, C.c_double, C.POINTER(abi.OdeControls), C.c_int,
                                             C.POINTER(C.c_double), C.POINTER(C.c_int)]
            lib.odo_locate_secant.restype = C.c_int
            lib.odo_locate_secant.argtypes = [C.POINTER(abi.Model), C.c_int, C.c_double, C.c_void_p, C.c_void_p,
                                              C.c_double, C.c_int, C.c_double, C.c_double, C.c_double, C.c_void_p,
                                              C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_int)]
            lib.odo_rhs.restype = C.c_int
            lib.odo_rhs_batch.restype = C.c_int
            lib.odo_rhs_batch.argtypes = [C.POINTER(abi.Model), abi.Index, C.c_void_p, C.c_void_p, C.c_void_p,
                                          abi.Index, abi.Index, C.c_void_p]
            lib.odo_rhs.argtypes = [C.POINTER(abi.Model), C.c_double, C.c_void_p, C.c_void_p, C.c_void_p]
        _libs[which] = lib
    return _libs[which]


class CheckerError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code
        self.msg = msg


def solve(which: str, model, td, y, p, acc, *, algorithm: int, dt: float, iterations: int = 1,
          outcomes: np.ndarray | None = None, trace: bool = False, workers: int = 1, tile_size: int = 64,
          ode=None):
    """Run `iterations` solves in place on flat SoA arrays. Returns
    (outcomes, seconds, trace_dict_or_None)."""
    lib = load(which)
    d = model.dims()
    n = td.size // 2
    keep = outcomes is not None
    if outcomes is None:
        outcomes = abi.empty_outcomes(n)
    cfg = abi.SolverConfig(algorithm, 0, dt, tile_size, workers)
    ode_c = (ode or model.ode_controls()).to_c()
    tr = None
    if trace:
        tr = dict(
            td=np.zeros(iterations * 2 * n),
            state=np.zeros(iterations * d.system_dim * n),
            acc=np.zeros(iterations * max(d.accessory_count, 1) * n),
            outcomes=np.zeros(iterations * n, dtype=abi.OUTCOME_DTYPE),
        )
    secs = C.c_double(0)
    fn = lib.odo_solve if which == "port" else lib.odref_solve
    rc = fn(C.byref(model.to_c()), n, abi.vptr(td), abi.vptr(y), abi.vptr(p if p.size else None),
            abi.vptr(acc if acc.size else None), abi.vptr(outcomes), int(keep), C.byref(cfg), C.byref(ode_c),
            iterations, abi.vptr(tr["td"]) if tr else None, abi.vptr(tr["state"]) if tr else None,
            abi.vptr(tr["acc"]) if tr else None, abi.vptr(tr["outcomes"]) if tr else None, C.byref(secs))
    if rc != 0:
        err = (lib.odo_last_error() if which == "port" else lib.odref_last_error()).decode()
        raise CheckerError(rc, err)
    return outcomes, secs.value, tr


def reference_detections(wl, iterations: int = 1, workers: int = 4):
    """Run the reference (oracle/_ref) on a workload with its own
    on_detection observer attached (solve.hpp:46-50): the last solve's
    detections as (records [abi.DETECTION_DTYPE], y_pre, y_post) in
    (system, call) order, plus the solve's result dict."""
    lib = load("reference")
    lib.odref_capture_detections.argtypes = [C.c_int]
    lib.odref_detections.restype = abi.Index
    lib.odref_detections.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, abi.Index]
    lib.odref_capture_detections(1)
    try:
        res = solve_workload("reference", wl, iterations, workers=workers)
        total = lib.odref_detections(None, None, None, 0)
        dim = wl.model.dims().system_dim
        rec = np.zeros(total, dtype=abi.DETECTION_DTYPE)
        pre, post = np.zeros((total, dim)), np.zeros((total, dim))
        if total:
            lib.odref_detections(abi.vptr(rec), abi.vptr(pre), abi.vptr(post), total)
    finally:
        lib.odref_capture_detections(0)
    return rec, pre, post, res


def solve_workload(which: str, wl, iterations: int | None = None, trace: bool = False, workers: int = 1):
    td, y, p, acc = wl.arrays()
    oc, secs, tr = solve(which, wl.model, td, y, p, acc, algorithm=wl.algorithm, dt=wl.dt,
                         iterations=iterations or wl.iterations, trace=trace, workers=workers)
    return dict(td=td, y=y, p=p, acc=acc, outcomes=oc, seconds=secs, trace=tr)


def scan(protocol: int, spec, workers: int = 0):
    """The reference's scan protocol (src/scan.cpp) on the same C spec as
    odegpu_scan_run: (rows, diagnostics dict)."""
    from paper_1810_03931_b200 import scan as gscan

    lib = load("reference")
    f = lib.odref_scan_run
    f.restype = C.c_int
    f.argtypes = [C.c_int32, C.c_void_p, C.POINTER(C.c_double), abi.Index, C.POINTER(abi.Index),
                  C.POINTER(abi.Index), C.POINTER(abi.ScanDiagnosticsC), C.c_int]
    cols = gscan.COLUMNS[protocol]
    rows = np.zeros((gscan.expected_rows(protocol, spec), len(cols)))
    nr, nc, d = abi.Index(), abi.Index(), abi.ScanDiagnosticsC()
    c_spec = spec.to_c()
    rc = f(protocol, C.byref(c_spec), rows.ctypes.data_as(C.POINTER(C.c_double)), rows.shape[0], C.byref(nr),
           C.byref(nc), C.byref(d), workers or host_cores())
    if rc != 0:
        raise CheckerError(rc, lib.odref_last_error().decode())
    return rows[: nr.value], gscan.diagnostics_dict(d)


def host_cores() -> int:
    return len(os.sched_getaffinity(0))
