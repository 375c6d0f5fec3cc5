"""ctypes mirror of include/odegpu.h (the C ABI of libodegpu).

Only plain structs and the loader live here. The library is built in-tree by
``__graft_entry__.build()`` (``paper_1810_03931_b200/lib/libodegpu.so``); on a
machine with a GPU a missing library is an error — there is no fallback path.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

PKG_DIR = Path(__file__).resolve().parent
LIB_DIR = PKG_DIR / "lib"
LIB_PATH = LIB_DIR / "libodegpu.so"
# the exact-parity build (make parity: -fmad=false, libdevice pow in the
# step controller); selected with ODEGPU_BUILD=parity or ODEGPU_LIB=<path>
PARITY_LIB_PATH = LIB_DIR / "libodegpu_parity.so"
BUILD_PARITY = 1  # odegpu_build_flags() bit

# include/odegpu.h constants
OK = 0
ERR_INVALID_ARGUMENT = -1
ERR_OUT_OF_RANGE = -2
ERR_CUDA = -3
ERR_UNSUPPORTED = -4

RK4, RKCK45 = 0, 1
FETCH_NATURAL, FETCH_COST, FETCH_AUTO = 0, 1, 2  # odegpu_batch_set_fetch_order
REACHED_END_TIME, EVENT_STOP, EQUILIBRIUM_STOP, NONFINITE_ABORT = 0, 1, 2, 3
COPY_TIME_DOMAIN, COPY_ACTUAL_STATE, COPY_PARAMETER, COPY_ACCESSORIES, COPY_ALL = 0, 1, 2, 3, 4
PROP_TIME_DOMAIN, PROP_STATE, PROP_PARAMETERS, PROP_ACCESSORIES = 0, 1, 2, 3

MODEL_DUFFING = 0
MODEL_DUFFING_MAX_ACCESSORY = 1
MODEL_DUFFING_MAX_EVENT = 2
MODEL_DUFFING_MAXMIN = 3
MODEL_KELLER_MIKSIS = 4
MODEL_BUBBLE_COLLAPSE = 5
MODEL_VALVE = 6
MODEL_DUFFING_LYAPUNOV = 7
MODEL_CONSTANT = 16
MODEL_CUBIC_TIME = 17
MODEL_EXPONENTIAL = 18
MODEL_UNIT_SLOPE = 19
MODEL_COUNTING = 20
MODEL_RAMP = 21
MODEL_DECAY = 22
MODEL_SEAT_CONTACT = 23
MODEL_HARMONIC = 24
MODEL_BLOWUP = 25

MAX_MODEL_CONSTS = 8

Index = C.c_int64


class Model(C.Structure):
    _fields_ = [("id", C.c_int32), ("reserved", C.c_int32), ("consts", C.c_double * MAX_MODEL_CONSTS)]


class SystemDims(C.Structure):
    _fields_ = [("system_dim", Index), ("param_count", Index), ("event_count", Index), ("accessory_count", Index)]


class PoolDims(C.Structure):
    _fields_ = [("problem_size", Index), ("system_dim", Index), ("param_count", Index), ("accessory_count", Index)]


class BatchDims(C.Structure):
    _fields_ = [
        ("batch_capacity", Index),
        ("system_dim", Index),
        ("param_count", Index),
        ("event_count", Index),
        ("accessory_count", Index),
    ]


class PoolView(C.Structure):
    _fields_ = [
        ("dims", PoolDims),
        ("time_domain", C.POINTER(C.c_double)),
        ("state", C.POINTER(C.c_double)),
        ("parameters", C.POINTER(C.c_double)),
        ("accessories", C.POINTER(C.c_double)),
    ]


class LinearCopySpec(C.Structure):
    _fields_ = [
        ("start_in_batch", Index),
        ("start_in_pool", Index),
        ("element_count", Index),
        ("copy_mode", C.c_int32),
        ("reserved", C.c_int32),
    ]


class SolverConfig(C.Structure):
    _fields_ = [
        ("algorithm", C.c_int32),
        ("reserved", C.c_int32),
        ("initial_time_step", C.c_double),
        ("tile_size", Index),
        ("worker_count", Index),
    ]


class OdeControls(C.Structure):
    _fields_ = [
        ("rel_tol", C.POINTER(C.c_double)),
        ("abs_tol", C.POINTER(C.c_double)),
        ("max_step", C.c_double),
        ("min_step", C.c_double),
        ("step_grow_limit", C.c_double),
        ("step_shrink_limit", C.c_double),
    ]


class EventControls(C.Structure):
    _fields_ = [
        ("direction", C.POINTER(C.c_int32)),
        ("tolerance", C.POINTER(C.c_double)),
        ("stop_condition", C.POINTER(Index)),
        ("max_steps_in_zone", Index),
    ]


# odegpu_detection: one record of the detection log (the reference's
# on_detection observer: Detection, events.hpp:40-47), 56 bytes.
DETECTION_DTYPE = np.dtype(
    {
        "names": ["system", "event_index", "counter", "sequence", "t", "value", "kind", "in_zone"],
        "formats": ["<i8", "<i8", "<i8", "<i8", "<f8", "<f8", "<i4", "<i4"],
        "offsets": [0, 8, 16, 24, 32, 40, 48, 52],
        "itemsize": 56,
    }
)
DETECTION_KINDS = ("SteppedAcross", "EnteredFromAbove", "EnteredFromBelow")  # events.hpp:31

# odegpu_outcome / odensemble::SystemOutcome (driver.hpp:34-42), 56 bytes.
OUTCOME_DTYPE = np.dtype(
    {
        "names": [
            "final_t",
            "reason",
            "accepted_steps",
            "rejected_steps",
            "event_detections",
            "secant_failures",
            "smallest_step",
        ],
        "formats": ["<f8", "u1", "<i8", "<i8", "<i8", "<i8", "<f8"],
        "offsets": [0, 8, 16, 24, 32, 40, 48],
        "itemsize": 56,
    }
)

class Diagnostics(C.Structure):
    _fields_ = [
        ("accepted_steps", Index),
        ("rejected_steps", Index),
        ("event_detections", Index),
        ("secant_failures", Index),
        ("reason_counts", Index * 4),
        ("max_trial_steps", Index),
    ]


class ChunkRecord(C.Structure):
    _fields_ = [
        ("td", C.POINTER(C.c_double)),
        ("state", C.POINTER(C.c_double)),
        ("accessories", C.POINTER(C.c_double)),
        ("outcomes", C.c_void_p),
    ]


class PoolOut(C.Structure):
    _fields_ = [
        ("time_domain", C.POINTER(C.c_double)),
        ("state", C.POINTER(C.c_double)),
        ("accessories", C.POINTER(C.c_double)),
        ("outcomes", C.c_void_p),
    ]


SINK = C.CFUNCTYPE(C.c_int, Index, C.c_void_p, C.c_void_p)
CHUNK_SINK = C.CFUNCTYPE(C.c_int, Index, Index, Index, C.POINTER(ChunkRecord), C.c_void_p)


def dptr(a: np.ndarray | None):
    if a is None:
        return C.POINTER(C.c_double)()
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(C.POINTER(C.c_double))


def vptr(a: np.ndarray | None):
    if a is None:
        return C.c_void_p()
    assert a.flags.c_contiguous
    return C.c_void_p(a.ctypes.data)


def empty_outcomes(n: int) -> np.ndarray:
    o = np.zeros(n, dtype=OUTCOME_DTYPE)
    o["smallest_step"] = np.inf
    return o


class LibraryMissing(RuntimeError):
    pass


# ---- scan protocols (include/odegpu.h: odegpu_scan_run)
SCAN_DUFFING_POINCARE, SCAN_DUFFING_MAXIMA_ACCESSORY, SCAN_DUFFING_MAXIMA_EVENT = 0, 1, 2
SCAN_DUFFING_LYAPUNOV, SCAN_BUBBLE, SCAN_VALVE = 3, 4, 5


class ParamRangeC(C.Structure):
    _fields_ = [("min", C.c_double), ("max", C.c_double), ("res", Index), ("log_scale", C.c_int32),
                ("reserved", C.c_int32)]


class ScanOptions(C.Structure):
    _fields_ = [("algorithm", C.c_int32), ("device", C.c_int32), ("dt", C.c_double), ("rel_tol", C.c_double),
                ("abs_tol", C.c_double), ("event_tol", C.c_double), ("batch_capacity", Index),
                ("devices", C.POINTER(C.c_int32)), ("n_devices", C.c_int32), ("reserved", C.c_int32)]


class DuffingScanC(C.Structure):
    _fields_ = [("k", ParamRangeC), ("forcing_amplitude", C.c_double), ("stiffness", C.c_double),
                ("forcing_omega", C.c_double), ("ic", C.c_double * 2), ("transient", Index), ("saved", Index),
                ("solver", ScanOptions)]


class BubbleScanC(C.Structure):
    _fields_ = [("pa1_bar", ParamRangeC), ("pa2_bar", ParamRangeC), ("f1_khz", ParamRangeC), ("f2_khz", ParamRangeC),
                ("R_E", C.c_double), ("c_L", C.c_double), ("rho_L", C.c_double), ("P_inf", C.c_double),
                ("p_V", C.c_double), ("sigma", C.c_double), ("mu_L", C.c_double), ("gamma", C.c_double),
                ("theta", C.c_double), ("ic", C.c_double * 2), ("t_end", C.c_double), ("transient", Index),
                ("saved", Index), ("solver", ScanOptions)]


class ValveScanC(C.Structure):
    _fields_ = [("q", ParamRangeC), ("kappa", C.c_double), ("delta", C.c_double), ("beta", C.c_double),
                ("restitution", C.c_double), ("ic", C.c_double * 3), ("t_end", C.c_double), ("transient", Index),
                ("saved", Index), ("solver", ScanOptions)]


class ScanDiagnosticsC(C.Structure):
    _fields_ = [("detections", Index), ("detections_outside_zone", Index), ("max_residual_ratio", C.c_double),
                ("secant_failures", Index), ("nonfinite_systems", Index), ("reason_counts", Index * 4),
                ("start_times_strictly_increase", C.c_int32), ("reserved", C.c_int32)]


class ScanTally(C.Structure):
    _fields_ = [("reason_counts", Index * 4), ("secant_failures", Index), ("detections", Index),
                ("detections_outside_zone", Index), ("max_residual_ratio", C.c_double),
                ("start_time_not_advanced", Index), ("nonfinite_systems", Index)]


_lib = None


def _bind(lib):
    P = C.POINTER
    vp = C.c_void_p
    sig = {
        "odegpu_abi_version": (C.c_int, []),
        "odegpu_build_flags": (C.c_int, []),
        "odegpu_last_error": (C.c_char_p, []),
        "odegpu_device_count": (C.c_int, []),
        "odegpu_model_dims": (C.c_int, [P(Model), P(SystemDims)]),
        "odegpu_batch_create": (C.c_int, [P(BatchDims), C.c_int, P(vp)]),
        "odegpu_batch_destroy": (None, [vp]),
        "odegpu_batch_dims_get": (C.c_int, [vp, P(BatchDims)]),
        "odegpu_batch_set_stream": (C.c_int, [vp, vp]),
        "odegpu_batch_set_fetch_order": (C.c_int, [vp, C.c_int32]),
        "odegpu_linear_set": (C.c_int, [vp, P(PoolView), P(LinearCopySpec)]),
        "odegpu_random_set": (C.c_int, [vp, P(PoolView), P(Index), P(Index), Index, C.c_int32]),
        "odegpu_batch_read": (C.c_int, [vp, C.c_int32, P(C.c_double)]),
        "odegpu_batch_write": (C.c_int, [vp, C.c_int32, P(C.c_double)]),
        "odegpu_batch_read_range": (C.c_int, [vp, C.c_int32, Index, Index, P(C.c_double), Index]),
        "odegpu_batch_write_range": (C.c_int, [vp, C.c_int32, Index, Index, P(C.c_double), Index]),
        "odegpu_batch_read_outcomes": (C.c_int, [vp, vp]),
        "odegpu_batch_write_outcomes": (C.c_int, [vp, vp]),
        "odegpu_batch_reset_outcomes": (C.c_int, [vp]),
        "odegpu_solve": (C.c_int, [vp, P(Model), P(SolverConfig), P(OdeControls), P(EventControls)]),
        "odegpu_solve_iteratively": (
            C.c_int,
            [vp, P(Model), P(SolverConfig), P(OdeControls), P(EventControls), Index, SINK, vp],
        ),
        "odegpu_batch_sync": (C.c_int, [vp]),
        "odegpu_batch_launch_count": (C.c_int64, [vp]),
        "odegpu_batch_set_detection_log": (C.c_int, [vp, Index]),
        "odegpu_batch_device": (C.c_int, [vp]),
        "odegpu_device_pool_create": (C.c_int, [P(PoolDims), C.c_int, P(vp)]),
        "odegpu_device_pool_destroy": (None, [vp]),
        "odegpu_device_pool_write": (C.c_int, [vp, C.c_int32, Index, Index, P(C.c_double), Index]),
        "odegpu_device_pool_read": (C.c_int, [vp, C.c_int32, Index, Index, P(C.c_double), Index]),
        "odegpu_device_pool_read_outcomes": (C.c_int, [vp, Index, Index, vp]),
        "odegpu_linear_set_device": (C.c_int, [vp, vp, P(LinearCopySpec)]),
        "odegpu_random_set_device": (C.c_int, [vp, vp, P(Index), P(Index), Index, C.c_int32]),
        "odegpu_device_pool_store": (C.c_int, [vp, vp, P(Index), P(Index), Index, C.c_int32]),
        "odegpu_device_pool_solve": (C.c_int, [vp, P(Model), P(SolverConfig), P(OdeControls), P(EventControls),
                                               Index, Index, C.c_int32]),
        "odegpu_model_keeps_time_domain": (C.c_int, [P(Model), P(C.c_int)]),
        "odegpu_batch_read_detection_log": (C.c_int, [vp, vp, P(C.c_double), P(C.c_double), Index, P(Index),
                                                      P(Index)]),
        "odegpu_batch_diagnostics": (C.c_int, [vp, P(Diagnostics)]),
        "odegpu_batch_last_kernel_ms": (C.c_int, [vp, P(C.c_double)]),
        "odegpu_batch_trial_steps": (C.c_int, [vp, P(Index), C.c_int]),
        "odegpu_batch_trig_certified": (C.c_int, [vp, P(C.c_int)]),
        "odegpu_dfma_peak": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, P(C.c_double), P(C.c_double)]),
        "odegpu_batch_copy": (C.c_int, [vp, vp]),
        "odegpu_solve_pool": (
            C.c_int,
            [P(PoolView), P(PoolOut), P(Model), P(SolverConfig), P(OdeControls), P(EventControls), Index, Index,
             Index, C.c_uint32, CHUNK_SINK, vp, C.c_int],
        ),
        "odegpu_solve_pool_multi": (
            C.c_int,
            [P(PoolView), P(PoolOut), P(Model), P(SolverConfig), P(OdeControls), P(EventControls), Index, Index,
             Index, C.c_uint32, CHUNK_SINK, vp, P(C.c_int), C.c_int],
        ),
        "odegpu_pipeline_create": (C.c_int, [P(Model), Index, C.c_int, P(vp)]),
        "odegpu_pipeline_run": (
            C.c_int,
            [vp, P(PoolView), P(PoolOut), P(SolverConfig), P(OdeControls), P(EventControls), Index, Index,
             C.c_uint32, CHUNK_SINK, vp],
        ),
        "odegpu_pipeline_destroy": (None, [vp]),
        "odegpu_pipeline_set_mode": (C.c_int, [vp, C.c_int32]),
        "odegpu_pipeline_last_mode": (C.c_int, [vp, P(C.c_int32)]),
        "odegpu_pipeline_run_tallied": (
            C.c_int,
            [vp, P(PoolView), P(PoolOut), P(SolverConfig), P(OdeControls), P(EventControls), Index, Index,
             C.c_uint32, CHUNK_SINK, vp, P(ScanTally)],
        ),
        "odegpu_scan_run": (C.c_int, [C.c_int32, vp, P(C.c_double), Index, P(Index), P(Index), P(ScanDiagnosticsC),
                                      C.c_char_p]),
        "odegpu_solve_pool_multi_tallied": (
            C.c_int,
            [P(PoolView), P(PoolOut), P(Model), P(SolverConfig), P(OdeControls), P(EventControls), Index, Index,
             Index, C.c_uint32, CHUNK_SINK, vp, P(C.c_int), C.c_int, C.c_int, P(ScanTally)],
        ),
        "odegpu_param_range_values": (C.c_int, [P(ParamRangeC), P(C.c_double)]),
        "odegpu_math_check": (C.c_int, [C.c_int, Index, vp, vp, vp, vp]),
        "odegpu_slice": (C.c_int, [Index, C.c_int, C.c_int, P(Index), P(Index)]),
        "odegpu_host_register": (C.c_int, [vp, C.c_size_t]),
        "odegpu_host_unregister": (C.c_int, [vp]),
    }
    # an older tuning variant (ODEGPU_LIB=lib/variants/*.so, A/B runs) may
    # lack newer entry points; the in-tree library must export them all
    variant = "variants" in Path(os.environ.get("ODEGPU_LIB", "")).parts
    for name, (res, args) in sig.items():
        if variant and not hasattr(lib, name):
            continue
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


def exported_symbols() -> list[str]:
    """Every function include/odegpu.h declares (parsed from the header)."""
    import re

    hdr = (PKG_DIR.parent / "include" / "odegpu.h").read_text()
    return sorted(set(re.findall(r"^\w[\w\s\*]*?\b(odegpu_\w+)\s*\(", hdr, flags=re.M)))


def load() -> C.CDLL:
    """Load the in-tree libodegpu.so (fails loudly if it was not built)."""
    global _lib
    if _lib is None:
        default = PARITY_LIB_PATH if os.environ.get("ODEGPU_BUILD") == "parity" else LIB_PATH
        path = Path(os.environ.get("ODEGPU_LIB", default))
        if not path.exists():
            raise LibraryMissing(
                f"{path} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            )
        _lib = _bind(C.CDLL(str(path)))
    return _lib
