"""Python mirror of the reference's pool / batch / solve API over the C ABI.

Same names, argument meaning and error behaviour as
/root/reference/proj/include/odensemble/{pool,batch,solve}.hpp, so parity
tests read like the reference's own tests. All compute goes through
libodegpu (include/odegpu.h); there is no CPU path here.

Errors: the reference's std::invalid_argument maps to InvalidArgument
(a ValueError), std::out_of_range to OutOfRange (an IndexError).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import weakref

import numpy as np

from . import abi
from .models import SystemDef, SystemDims


class OdegpuError(RuntimeError):
    code = abi.ERR_CUDA


class InvalidArgument(OdegpuError, ValueError):
    code = abi.ERR_INVALID_ARGUMENT


class OutOfRange(OdegpuError, IndexError):
    code = abi.ERR_OUT_OF_RANGE


class Unsupported(OdegpuError):
    code = abi.ERR_UNSUPPORTED


_ERRORS = {abi.ERR_INVALID_ARGUMENT: InvalidArgument, abi.ERR_OUT_OF_RANGE: OutOfRange,
           abi.ERR_UNSUPPORTED: Unsupported}


def check(rc: int):
    if rc != 0:
        msg = abi.load().odegpu_last_error().decode()
        raise _ERRORS.get(rc, OdegpuError)(msg)


Algorithm_RK4, Algorithm_RKCK45 = abi.RK4, abi.RKCK45


@dataclass
class SolverConfig:
    """driver.hpp:25-30."""

    algorithm: int = abi.RKCK45
    initial_time_step: float = 1e-3
    tile_size: int = 64
    worker_count: int = 1

    def to_c(self):
        return abi.SolverConfig(self.algorithm, 0, self.initial_time_step, self.tile_size, self.worker_count)


@dataclass
class PoolDims:
    problem_size: int
    system_dim: int
    param_count: int
    accessory_count: int

    def validate(self):  # pool.hpp:51-56
        if self.problem_size < 1:
            raise InvalidArgument("PoolDims: problem_size must be >= 1")
        if self.system_dim < 1:
            raise InvalidArgument("PoolDims: system_dim must be >= 1")
        if self.param_count < 0:
            raise InvalidArgument("PoolDims: param_count must be >= 0")
        if self.accessory_count < 0:
            raise InvalidArgument("PoolDims: accessory_count must be >= 0")


@dataclass
class BatchDims:
    batch_capacity: int
    system_dim: int
    param_count: int
    event_count: int
    accessory_count: int

    def to_c(self):
        return abi.BatchDims(self.batch_capacity, self.system_dim, self.param_count, self.event_count,
                             self.accessory_count)


def make_batch_dims(capacity: int, sys: SystemDims) -> BatchDims:
    """pool.hpp:65-69."""
    return BatchDims(capacity, sys.system_dim, sys.param_count, sys.event_count, sys.accessory_count)


def flat_index(idx: int, component: int, count: int) -> int:
    """pool.hpp:16-23."""
    if idx < 0 or idx >= count:
        raise OutOfRange(f"flat_index: system index {idx} outside [0, {count})")
    if component < 0:
        raise OutOfRange("flat_index: negative component index")
    return idx + component * count


class ProblemPool:
    """Host pool in SoA layout (pool.hpp:74-139). Arrays are numpy views."""

    def __init__(self, dims: PoolDims):
        dims.validate()
        self.dims = dims
        n = dims.problem_size
        self._td = np.zeros(2 * n)
        self._state = np.zeros(dims.system_dim * n)
        self._params = np.zeros(dims.param_count * n)
        self._acc = np.zeros(dims.accessory_count * n)

    def size(self):
        return self.dims.problem_size

    def time_domain(self):
        return self._td

    def state(self):
        return self._state

    def parameters(self):
        return self._params

    def accessories(self):
        return self._acc

    def _check(self, c, count, what):
        if c < 0 or c >= count:
            raise OutOfRange(f"ProblemPool: {what} component out of range")

    def set_time(self, idx, t0, t1):
        n = self.size()
        self._td[flat_index(idx, 0, n)] = t0
        self._td[flat_index(idx, 1, n)] = t1

    def time_start(self, idx):
        return self._td[flat_index(idx, 0, self.size())]

    def time_end(self, idx):
        return self._td[flat_index(idx, 1, self.size())]

    def state_at(self, idx, c):
        self._check(c, self.dims.system_dim, "state")
        return self._state[flat_index(idx, c, self.size())]

    def set_state(self, idx, c, v):
        self._check(c, self.dims.system_dim, "state")
        self._state[flat_index(idx, c, self.size())] = v

    def param_at(self, idx, c):
        self._check(c, self.dims.param_count, "parameter")
        return self._params[flat_index(idx, c, self.size())]

    def set_param(self, idx, c, v):
        self._check(c, self.dims.param_count, "parameter")
        self._params[flat_index(idx, c, self.size())] = v

    def accessory_at(self, idx, c):
        self._check(c, self.dims.accessory_count, "accessory")
        return self._acc[flat_index(idx, c, self.size())]

    def set_accessory(self, idx, c, v):
        self._check(c, self.dims.accessory_count, "accessory")
        self._acc[flat_index(idx, c, self.size())] = v

    def view(self):
        v = abi.PoolView(
            abi.PoolDims(self.dims.problem_size, self.dims.system_dim, self.dims.param_count,
                         self.dims.accessory_count),
            abi.dptr(self._td), abi.dptr(self._state), abi.dptr(self._params if self._params.size else None),
            abi.dptr(self._acc if self._acc.size else None))
        v._keep = self
        return v

    def pin(self) -> "ProblemPool":
        """Moves the pool's arrays into page-locked host memory (pinned()),
        so pipeline copies are asynchronous and the streaming mode applies."""
        self._td, self._state, self._params, self._acc = (pinned(a) for a in (self._td, self._state, self._params,
                                                                                  self._acc))
        return self

    @staticmethod
    def from_arrays(td, y, p, acc) -> "ProblemPool":
        """Pool over flat SoA arrays (copied)."""
        n = td.size // 2
        pool = ProblemPool(PoolDims(n, y.size // n, p.size // n, acc.size // n))
        pool._td[:] = td
        pool._state[:] = y
        pool._params[:] = p
        pool._acc[:] = acc
        return pool


# CopyMode (pool.hpp:142)
class CopyMode:
    TimeDomain, ActualState, Parameter, Accessories, All = (abi.COPY_TIME_DOMAIN, abi.COPY_ACTUAL_STATE,
                                                            abi.COPY_PARAMETER, abi.COPY_ACCESSORIES, abi.COPY_ALL)


@dataclass
class LinearCopySpec:
    start_in_batch: int = 0
    start_in_pool: int = 0
    element_count: int = 0
    copy_mode: int = CopyMode.All


@dataclass
class RandomCopySpec:
    indices_in_batch: list
    indices_in_pool: list
    copy_mode: int = CopyMode.All


class SolverBatch:
    """Device-resident batch (batch.hpp:17-67) on one GPU. Accessors copy the
    device arrays back (D2H) — the lazy host mirror of the reference's
    spans."""

    def __init__(self, dims: BatchDims, device: int = 0):
        self._lib = abi.load()
        self.dims = dims
        self.device = device
        h = C.c_void_p()
        check(self._lib.odegpu_batch_create(C.byref(dims.to_c()), device, C.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            self._lib.odegpu_batch_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def size(self):
        return self.dims.batch_capacity

    def _read(self, prop, comps):
        out = np.zeros(comps * self.size())
        if comps:
            check(self._lib.odegpu_batch_read(self._h, prop, abi.dptr(out)))
        return out

    def _write(self, prop, arr):
        arr = np.ascontiguousarray(arr, dtype=np.float64)
        check(self._lib.odegpu_batch_write(self._h, prop, abi.dptr(arr)))

    def time_domain(self):
        return self._read(abi.PROP_TIME_DOMAIN, 2)

    def state(self):
        return self._read(abi.PROP_STATE, self.dims.system_dim)

    def parameters(self):
        return self._read(abi.PROP_PARAMETERS, self.dims.param_count)

    def accessories(self):
        return self._read(abi.PROP_ACCESSORIES, self.dims.accessory_count)

    def set_time_domain(self, a):
        self._write(abi.PROP_TIME_DOMAIN, a)

    def set_state(self, a):
        self._write(abi.PROP_STATE, a)

    def set_parameters(self, a):
        self._write(abi.PROP_PARAMETERS, a)

    def set_accessories(self, a):
        self._write(abi.PROP_ACCESSORIES, a)

    def outcomes(self) -> np.ndarray:
        out = np.zeros(self.size(), dtype=abi.OUTCOME_DTYPE)
        check(self._lib.odegpu_batch_read_outcomes(self._h, abi.vptr(out)))
        return out

    def set_outcomes(self, o: np.ndarray):
        o = np.ascontiguousarray(o, dtype=abi.OUTCOME_DTYPE)
        check(self._lib.odegpu_batch_write_outcomes(self._h, abi.vptr(o)))

    def reset_outcomes(self):
        check(self._lib.odegpu_batch_reset_outcomes(self._h))

    def time_start(self, i):
        return self.time_domain()[flat_index(i, 0, self.size())]

    def time_end(self, i):
        return self.time_domain()[flat_index(i, 1, self.size())]

    def state_at(self, i, c):
        return self.state()[flat_index(i, c, self.size())]

    def param_at(self, i, c):
        return self.parameters()[flat_index(i, c, self.size())]

    def accessory_at(self, i, c):
        return self.accessories()[flat_index(i, c, self.size())]

    def set_stream(self, stream_handle: int | None):
        check(self._lib.odegpu_batch_set_stream(self._h, C.c_void_p(stream_handle or 0)))

    def set_fetch_order(self, mode: int):
        """abi.FETCH_NATURAL / FETCH_COST / FETCH_AUTO (odegpu_batch_set_fetch_order)."""
        check(self._lib.odegpu_batch_set_fetch_order(self._h, mode))

    def sync(self):
        check(self._lib.odegpu_batch_sync(self._h))

    def launch_count(self) -> int:
        return int(self._lib.odegpu_batch_launch_count(self._h))

    def set_detection_log(self, capacity: int):
        """Record every detection of the following solves (the reference's
        on_detection observer, solve.hpp:46-50); 0 disables the log."""
        check(self._lib.odegpu_batch_set_detection_log(self._h, int(capacity)))

    def detection_log(self, capacity: int | None = None):
        """The last solve's detections ordered by (system, sequence):
        (records [abi.DETECTION_DTYPE], y_pre [k, dim], y_post [k, dim], total)."""
        dim = self.dims.system_dim
        cnt, tot = C.c_int64(), C.c_int64()
        check(self._lib.odegpu_batch_read_detection_log(self._h, None, None, None, 0, C.byref(cnt), C.byref(tot)))
        k = min(int(tot.value), capacity if capacity is not None else int(tot.value))
        rec = np.zeros(k, dtype=abi.DETECTION_DTYPE)
        pre = np.zeros((k, dim))
        post = np.zeros((k, dim))
        if k:
            dp = C.POINTER(C.c_double)
            check(self._lib.odegpu_batch_read_detection_log(self._h, rec.ctypes.data_as(C.c_void_p),
                                                            pre.ctypes.data_as(dp), post.ctypes.data_as(dp),
                                                            k, C.byref(cnt), C.byref(tot)))
            rec, pre, post = rec[: cnt.value], pre[: cnt.value], post[: cnt.value]
        return rec, pre, post, int(tot.value)

    def diagnostics(self) -> dict:
        """Device-side tally of the last solve's outcomes."""
        d = abi.Diagnostics()
        check(self._lib.odegpu_batch_diagnostics(self._h, C.byref(d)))
        return dict(accepted_steps=d.accepted_steps, rejected_steps=d.rejected_steps,
                    event_detections=d.event_detections, secant_failures=d.secant_failures,
                    reason_counts=list(d.reason_counts), max_trial_steps=d.max_trial_steps)

    def trig_certified(self) -> bool:
        """Whether the last solve ran the certified (branch-free trig) path."""
        v = C.c_int()
        check(self._lib.odegpu_batch_trig_certified(self._h, C.byref(v)))
        return bool(v.value)

    def trial_steps(self, reset: bool = False) -> int:
        """Trial steps the batch's solve kernels integrated since creation or
        the last reset (every system and iteration, fused ones included)."""
        v = C.c_int64()
        check(self._lib.odegpu_batch_trial_steps(self._h, C.byref(v), int(reset)))
        return int(v.value)

    def last_kernel_ms(self) -> float:
        v = C.c_double()
        check(self._lib.odegpu_batch_last_kernel_ms(self._h, C.byref(v)))
        return v.value


def linear_set(batch: SolverBatch, pool: ProblemPool, spec: LinearCopySpec):
    """batch.cpp:78-104."""
    c = abi.LinearCopySpec(spec.start_in_batch, spec.start_in_pool, spec.element_count, spec.copy_mode, 0)
    check(batch._lib.odegpu_linear_set(batch.handle, C.byref(pool.view()), C.byref(c)))


def random_set(batch: SolverBatch, pool: ProblemPool, spec: RandomCopySpec):
    """batch.cpp:106-135."""
    ib = np.ascontiguousarray(spec.indices_in_batch, dtype=np.int64)
    ip = np.ascontiguousarray(spec.indices_in_pool, dtype=np.int64)
    if ib.size != ip.size:
        raise InvalidArgument("random_set: index lists differ in length")
    P = C.POINTER(C.c_int64)
    check(batch._lib.odegpu_random_set(batch.handle, C.byref(pool.view()), ib.ctypes.data_as(P),
                                       ip.ctypes.data_as(P), ib.size, spec.copy_mode))


class DevicePool:
    """A ProblemPool (pool.hpp:12-64) kept in HBM (odegpu_device_pool_*):
    linear_set / random_set from it are device gathers; solve() runs the
    whole pool in chunks, cost-clustered on request."""

    def __init__(self, dims: PoolDims, device: int = 0):
        dims.validate()
        self._lib = abi.load()
        self.dims = dims
        self.device = device
        h = C.c_void_p()
        check(self._lib.odegpu_device_pool_create(C.byref(abi.PoolDims(dims.problem_size, dims.system_dim,
                                                                         dims.param_count, dims.accessory_count)),
                                                  device, C.byref(h)))
        self._h = h

    @classmethod
    def from_pool(cls, pool: ProblemPool, device: int = 0) -> "DevicePool":
        dp = cls(pool.dims, device)
        dp.upload(pool)
        return dp

    @property
    def handle(self):
        return self._h

    def close(self):
        if getattr(self, "_h", None):
            self._lib.odegpu_device_pool_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _comps(self, prop):
        d = self.dims
        return {abi.PROP_TIME_DOMAIN: 2, abi.PROP_STATE: d.system_dim, abi.PROP_PARAMETERS: d.param_count,
                abi.PROP_ACCESSORIES: d.accessory_count}[prop]

    def write(self, prop: int, a: np.ndarray, start: int = 0, count: int | None = None):
        n = self.dims.problem_size if count is None else count
        a = np.ascontiguousarray(a, dtype=np.float64)
        if a.size != self._comps(prop) * n:
            raise InvalidArgument("device pool: array size != components x count")
        check(self._lib.odegpu_device_pool_write(self._h, prop, start, n, abi.dptr(a if a.size else None), n))

    def read(self, prop: int, start: int = 0, count: int | None = None) -> np.ndarray:
        n = self.dims.problem_size if count is None else count
        out = np.zeros(self._comps(prop) * n)
        check(self._lib.odegpu_device_pool_read(self._h, prop, start, n, abi.dptr(out if out.size else None), n))
        return out

    def upload(self, pool: ProblemPool):
        for prop, a in ((abi.PROP_TIME_DOMAIN, pool.time_domain()), (abi.PROP_STATE, pool.state()),
                        (abi.PROP_PARAMETERS, pool.parameters()), (abi.PROP_ACCESSORIES, pool.accessories())):
            if a.size:
                self.write(prop, a)

    def time_domain(self):
        return self.read(abi.PROP_TIME_DOMAIN)

    def state(self):
        return self.read(abi.PROP_STATE)

    def parameters(self):
        return self.read(abi.PROP_PARAMETERS)

    def accessories(self):
        return self.read(abi.PROP_ACCESSORIES)

    def outcomes(self) -> np.ndarray:
        o = np.zeros(self.dims.problem_size, dtype=abi.OUTCOME_DTYPE)
        check(self._lib.odegpu_device_pool_read_outcomes(self._h, 0, o.size, abi.vptr(o)))
        return o

    def solve(self, defn: SystemDef, cfg: SolverConfig | None = None, batch_capacity: int | None = None,
              iterations: int = 1, clustered: bool = True):
        """odegpu_device_pool_solve: every system `iterations` times in place."""
        m, c, ode, ev, _ = _prepared(defn, cfg or SolverConfig())
        cap = batch_capacity or self.dims.problem_size
        check(self._lib.odegpu_device_pool_solve(self._h, m, c, ode, ev, cap, iterations, int(bool(clustered))))

    def store(self, batch: SolverBatch, spec: RandomCopySpec):
        """Batch slots spec.indices_in_batch back into pool rows spec.indices_in_pool."""
        ib = np.ascontiguousarray(spec.indices_in_batch, dtype=np.int64)
        ip = np.ascontiguousarray(spec.indices_in_pool, dtype=np.int64)
        if ib.size != ip.size:
            raise InvalidArgument("store: index lists differ in length")
        Pt = C.POINTER(C.c_int64)
        check(self._lib.odegpu_device_pool_store(self._h, batch.handle, ib.ctypes.data_as(Pt), ip.ctypes.data_as(Pt),
                                                 ib.size, spec.copy_mode))


def linear_set_device(batch: SolverBatch, pool: DevicePool, spec: LinearCopySpec):
    """batch.cpp:78-104 from a device pool."""
    c = abi.LinearCopySpec(spec.start_in_batch, spec.start_in_pool, spec.element_count, spec.copy_mode, 0)
    check(batch._lib.odegpu_linear_set_device(batch.handle, pool.handle, C.byref(c)))


def random_set_device(batch: SolverBatch, pool: DevicePool, spec: RandomCopySpec):
    """batch.cpp:106-135 from a device pool."""
    ib = np.ascontiguousarray(spec.indices_in_batch, dtype=np.int64)
    ip = np.ascontiguousarray(spec.indices_in_pool, dtype=np.int64)
    if ib.size != ip.size:
        raise InvalidArgument("random_set: index lists differ in length")
    Pt = C.POINTER(C.c_int64)
    check(batch._lib.odegpu_random_set_device(batch.handle, pool.handle, ib.ctypes.data_as(Pt),
                                              ip.ctypes.data_as(Pt), ib.size, spec.copy_mode))


def _controls(defn: SystemDef):
    ode = defn.ode_controls().to_c()
    ev = defn.event_controls().to_c()
    return ode, ev


_PREPARED: dict = {}


def _prepared(defn: SystemDef, cfg: SolverConfig):
    """The C structs of one (model, controls, config), built once per distinct
    value: keyed on the values themselves, so mutating a model or config
    between solves is picked up."""
    o, e = defn.ode_controls(), defn.event_controls()
    key = (type(defn), defn.model_id, tuple(defn.consts), tuple(o.rel_tol), tuple(o.abs_tol), o.max_step,
           o.min_step, o.step_grow_limit, o.step_shrink_limit, tuple(e.direction), tuple(e.tolerance),
           tuple(e.stop_condition), e.max_steps_in_zone, cfg.algorithm, cfg.initial_time_step, cfg.tile_size,
           cfg.worker_count)
    hit = _PREPARED.get(key)
    if hit is None:
        if len(_PREPARED) > 64:
            _PREPARED.clear()
        ode, ev = o.to_c(), e.to_c()
        m, c = defn.to_c(), cfg.to_c()
        hit = _PREPARED[key] = (C.byref(m), C.byref(c), C.byref(ode), C.byref(ev), (m, c, ode, ev))
    return hit


def solve(batch: SolverBatch, defn: SystemDef, cfg: SolverConfig | None = None):
    """solve.hpp:60-128 — synchronous, in place."""
    m, c, ode, ev, _ = _prepared(defn, cfg or SolverConfig())
    check(batch._lib.odegpu_solve(batch.handle, m, c, ode, ev))


def solve_iteratively(batch: SolverBatch, defn: SystemDef, cfg: SolverConfig | None, iterations: int, sink=None):
    """solve.hpp:133-142. sink(iteration, batch) after each solve; with no
    sink the iterations run back to back on the device."""
    m, c, ode, ev, _ = _prepared(defn, cfg or SolverConfig())
    err = []

    def _sink(it, _h, _u):
        try:
            sink(int(it), batch)
            return 0
        except BaseException as e:  # propagate after the C loop unwinds
            err.append(e)
            return 1

    cb = abi.SINK(_sink) if sink else abi.SINK()
    rc = batch._lib.odegpu_solve_iteratively(batch.handle, m, c, ode, ev, int(iterations), cb, None)
    if err:
        raise err[0]
    check(rc)


def batch_copy(dst: SolverBatch, src: SolverBatch):
    """Device-to-device copy of every array and outcome (same dims)."""
    check(dst._lib.odegpu_batch_copy(dst.handle, src.handle))


def slice_range(total: int, parts: int, index: int) -> tuple[int, int]:
    """Contiguous [begin, end) owned by part `index` of `parts` (odegpu_slice)."""
    b, e = C.c_int64(), C.c_int64()
    check(abi.load().odegpu_slice(total, parts, index, C.byref(b), C.byref(e)))
    return b.value, e.value


RECORD_TD, RECORD_STATE, RECORD_ACC, RECORD_OUTCOMES = 1, 2, 8, 16


_PAGE = 4096


def pinned(a: np.ndarray) -> np.ndarray:
    """A page-locked copy of `a` (odegpu_host_register over page-aligned
    numpy storage of its own, unregistered when the copy is collected)."""
    a = np.asarray(a)
    nbytes = max(a.nbytes, 1)
    span = -(-nbytes // _PAGE) * _PAGE
    raw = np.empty(span + _PAGE, dtype=np.uint8)
    off = (-raw.ctypes.data) % _PAGE
    buf = raw[off:off + span]
    lib = abi.load()
    check(lib.odegpu_host_register(C.c_void_p(buf.ctypes.data), span))
    weakref.finalize(raw, lib.odegpu_host_unregister, C.c_void_p(buf.ctypes.data))
    out = buf[:a.nbytes].view(a.dtype).reshape(a.shape)
    out[...] = a
    return out


def _pool_out(defn, n, arrays=None):
    d = defn.dims()
    if arrays is None:
        arrays = (np.zeros(2 * n), np.zeros(d.system_dim * n), np.zeros(d.accessory_count * n),
                  np.zeros(n, dtype=abi.OUTCOME_DTYPE))
    out = abi.PoolOut(abi.dptr(arrays[0]), abi.dptr(arrays[1]), abi.dptr(arrays[2] if d.accessory_count else None),
                      abi.vptr(arrays[3]))
    return arrays, out


def _chunk_sink(defn, record_mask, on_chunk, err):
    d = defn.dims()

    def _sink(start, count, nrec, rec_p, _u):
        try:
            rec = rec_p.contents
            got = {}
            if record_mask & RECORD_TD:
                got["td"] = np.ctypeslib.as_array(rec.td, shape=(nrec * 2 * count,)).copy()
            if record_mask & RECORD_STATE:
                got["state"] = np.ctypeslib.as_array(rec.state, shape=(nrec * d.system_dim * count,)).copy()
            if record_mask & RECORD_ACC and d.accessory_count:
                got["acc"] = np.ctypeslib.as_array(rec.accessories, shape=(nrec * d.accessory_count * count,)).copy()
            if record_mask & RECORD_OUTCOMES:
                buf = (C.c_char * (nrec * count * abi.OUTCOME_DTYPE.itemsize)).from_address(rec.outcomes)
                got["outcomes"] = np.frombuffer(buf, dtype=abi.OUTCOME_DTYPE).copy()
            on_chunk(int(start), int(count), got)
            return 0
        except BaseException as e:
            err.append(e)
            return 1

    return abi.CHUNK_SINK(_sink) if on_chunk else abi.CHUNK_SINK()


PIPELINE_AUTO, PIPELINE_CHUNKED, PIPELINE_STREAMING = 0, 1, 2  # enum odegpu_pipeline_mode


class Pipeline:
    """Persistent pool pipeline (odegpu_pipeline_*), reused by every run().
    CHUNKED: device batches of `batch_capacity` systems, chunk k+1's H2D and
    chunk k-1's D2H overlap chunk k's kernels. STREAMING: the pool becomes
    resident while one persistent solve kernel runs over it, gated chunk by
    chunk on the copies. AUTO (the default) runs the chunked slots; STREAMING is opt-in."""

    def __init__(self, defn: SystemDef, batch_capacity: int, device: int = 0, mode: int = PIPELINE_AUTO):
        self._lib = abi.load()
        self.defn = defn
        h = C.c_void_p()
        check(self._lib.odegpu_pipeline_create(C.byref(defn.to_c()), batch_capacity, device, C.byref(h)))
        self._h = h
        if mode != PIPELINE_AUTO:
            self.set_mode(mode)

    def set_mode(self, mode: int):
        check(self._lib.odegpu_pipeline_set_mode(self._h, mode))

    def last_mode(self) -> int:
        m = C.c_int32()
        check(self._lib.odegpu_pipeline_last_mode(self._h, C.byref(m)))
        return m.value

    def close(self):
        if getattr(self, "_h", None):
            self._lib.odegpu_pipeline_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def run(self, pool: ProblemPool, cfg: SolverConfig | None, iterations: int, *, record_from: int | None = None,
            record_mask: int = 0, on_chunk=None, out_arrays=None):
        cfg = cfg or SolverConfig()
        ode, ev = _controls(self.defn)
        record_from = iterations if record_from is None else record_from
        arrays, out = _pool_out(self.defn, pool.size(), out_arrays)
        err = []
        cb = _chunk_sink(self.defn, record_mask, on_chunk, err)
        rc = self._lib.odegpu_pipeline_run(self._h, C.byref(pool.view()), C.byref(out), C.byref(cfg.to_c()),
                                           C.byref(ode), C.byref(ev), iterations, record_from,
                                           record_mask if on_chunk else 0, cb, None)
        if err:
            raise err[0]
        check(rc)
        return arrays


def solve_pool(pool: ProblemPool, defn: SystemDef, cfg: SolverConfig | None, batch_capacity: int, iterations: int,
               *, record_from: int | None = None, record_mask: int = 0, on_chunk=None, write_back: bool = True,
               devices=(0,)):
    """Chunked pool pipeline (odegpu_solve_pool[_multi]): the pool runs through
    the device(s) in chunks of `batch_capacity`, `iterations` solves each,
    with double-buffered copies. Returns (td, state, acc, outcomes) endpoint
    arrays (pool layout) if `write_back`. `on_chunk(start, count, records)`
    receives, per chunk, a dict of recorded per-iteration arrays."""
    cfg = cfg or SolverConfig()
    ode, ev = _controls(defn)
    n = pool.size()
    record_from = iterations if record_from is None else record_from
    out_arrays, out = _pool_out(defn, n) if write_back else (None, None)
    err = []
    cb = _chunk_sink(defn, record_mask, on_chunk, err)
    lib = abi.load()
    args = (C.byref(pool.view()), C.byref(out) if out is not None else None, C.byref(defn.to_c()),
            C.byref(cfg.to_c()), C.byref(ode), C.byref(ev), batch_capacity, iterations, record_from,
            record_mask if on_chunk else 0, cb, None)
    devices = list(devices)
    if len(devices) == 1:
        rc = lib.odegpu_solve_pool(*args, devices[0])
    else:
        dev_arr = (C.c_int * len(devices))(*devices)
        rc = lib.odegpu_solve_pool_multi(*args, dev_arr, len(devices))
    if err:
        raise err[0]
    check(rc)
    return out_arrays


def dfma_peak(device: int = 0, blocks: int | None = None, threads: int = 256, iters: int = 4096):
    """Lane-DFMA/s of the FP64 pipe measured by the microbenchmark kernel."""
    lib = abi.load()
    if blocks is None:
        blocks = 148 * 16
    rate, secs = C.c_double(), C.c_double()
    check(lib.odegpu_dfma_peak(device, blocks, threads, iters, C.byref(rate), C.byref(secs)))
    return rate.value, secs.value
