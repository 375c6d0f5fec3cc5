"""System definitions (the reference's SystemModel implementations) as seen
from the host: dimensions, ODE/event controls and the model descriptor the C
ABI takes. The hooks themselves are compiled into libodegpu
(include/odegpu/models/*.hpp); here only their host-side data lives.

Mirrors /root/reference/proj/include/odensemble/system.hpp:21-43 (controls)
and models/{duffing,keller_miksis,valve}.hpp (constructors and controls),
plus the fakes of the reference tests (tests/test_*.cpp) used as KATs.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import abi


@dataclass
class OdeControls:
    """system.hpp:21-35."""

    rel_tol: list[float]
    abs_tol: list[float]
    max_step: float = 1.0e6
    min_step: float = 1.0e-12
    step_grow_limit: float = 5.0
    step_shrink_limit: float = 0.1

    @staticmethod
    def uniform(system_dim: int, rel: float, abs_: float) -> "OdeControls":
        return OdeControls([rel] * system_dim, [abs_] * system_dim)

    def to_c(self):
        rel = np.ascontiguousarray(self.rel_tol, dtype=np.float64)
        ab = np.ascontiguousarray(self.abs_tol, dtype=np.float64)
        c = abi.OdeControls(
            abi.dptr(rel), abi.dptr(ab), self.max_step, self.min_step, self.step_grow_limit, self.step_shrink_limit
        )
        c._keep = (rel, ab)
        return c


@dataclass
class EventControls:
    """system.hpp:38-43."""

    direction: list[int] = field(default_factory=list)
    tolerance: list[float] = field(default_factory=list)
    stop_condition: list[int] = field(default_factory=list)
    max_steps_in_zone: int = 50

    def to_c(self):
        d = np.ascontiguousarray(self.direction, dtype=np.int32)
        t = np.ascontiguousarray(self.tolerance, dtype=np.float64)
        s = np.ascontiguousarray(self.stop_condition, dtype=np.int64)
        c = abi.EventControls(
            d.ctypes.data_as(C.POINTER(C.c_int32)),
            abi.dptr(t),
            s.ctypes.data_as(C.POINTER(C.c_int64)),
            self.max_steps_in_zone,
        )
        c._keep = (d, t, s)
        return c


@dataclass(frozen=True)
class SystemDims:
    """pool.hpp:58-63."""

    system_dim: int
    param_count: int
    event_count: int
    accessory_count: int


class SystemDef:
    """Host handle of one compiled SystemModel."""

    model_id: int = -1
    _dims: SystemDims

    def __init__(self, ode: OdeControls | None = None, consts=()):
        self.ode = ode
        self.consts = list(consts)

    def dims(self) -> SystemDims:
        return self._dims

    def ode_controls(self) -> OdeControls:
        return self.ode

    def event_controls(self) -> EventControls:
        return EventControls()

    def keeps_time_domain(self) -> bool:
        """Whether a solve never changes a time domain (hooks.hpp
        kKeepsTimeDomain; odegpu_model_keeps_time_domain)."""
        import ctypes as C

        v = C.c_int()
        rc = abi.load().odegpu_model_keeps_time_domain(C.byref(self.to_c()), C.byref(v))
        if rc != 0:
            raise RuntimeError(abi.load().odegpu_last_error().decode())
        return bool(v.value)

    def to_c(self) -> abi.Model:
        m = abi.Model()
        m.id = self.model_id
        for i, v in enumerate(self.consts):
            m.consts[i] = float(v)
        return m


# --------------------------------------------------------------- reference models


class DuffingSystem(SystemDef):
    """models/duffing.hpp:75-88."""

    model_id = abi.MODEL_DUFFING
    _dims = SystemDims(2, 4, 0, 0)

    def __init__(self, ode: OdeControls | None = None):
        super().__init__(ode or OdeControls.uniform(2, 1e-9, 1e-9))


class DuffingMaxAccessorySystem(SystemDef):
    """models/duffing.hpp:92-117."""

    model_id = abi.MODEL_DUFFING_MAX_ACCESSORY
    _dims = SystemDims(2, 4, 0, 2)

    def __init__(self, ode: OdeControls | None = None):
        super().__init__(ode or OdeControls.uniform(2, 1e-9, 1e-9))


class DuffingMaxEventSystem(SystemDef):
    """models/duffing.hpp:122-156."""

    model_id = abi.MODEL_DUFFING_MAX_EVENT
    _dims = SystemDims(2, 4, 1, 2)

    def __init__(self, event_tolerance: float = 1e-6, stop_after: int = 0, ode: OdeControls | None = None):
        super().__init__(ode or OdeControls.uniform(2, 1e-9, 1e-9), (event_tolerance, stop_after))
        self.tol, self.stop = event_tolerance, stop_after

    def event_controls(self):
        return EventControls([-1], [self.tol], [self.stop])


class DuffingMaxMinSystem(SystemDef):
    """cfg1 harness model: acc = [y1_max, t_max, y1_min, t_min]."""

    model_id = abi.MODEL_DUFFING_MAXMIN
    _dims = SystemDims(2, 4, 0, 4)

    def __init__(self, ode: OdeControls | None = None):
        super().__init__(ode or OdeControls.uniform(2, 1e-9, 1e-9))


class KellerMiksisSystem(SystemDef):
    """models/keller_miksis.hpp:106-119."""

    model_id = abi.MODEL_KELLER_MIKSIS
    _dims = SystemDims(2, 13, 0, 0)

    def __init__(self, ode: OdeControls | None = None):
        super().__init__(ode or OdeControls.uniform(2, 1e-10, 1e-10))


class BubbleCollapseSystem(SystemDef):
    """models/keller_miksis.hpp:126-165."""

    model_id = abi.MODEL_BUBBLE_COLLAPSE
    _dims = SystemDims(2, 13, 1, 4)

    def __init__(self, event_tolerance: float = 1e-6, ode: OdeControls | None = None):
        super().__init__(ode or OdeControls.uniform(2, 1e-10, 1e-10), (event_tolerance,))
        self.tol = event_tolerance

    def event_controls(self):
        return EventControls([-1], [self.tol], [1])


class ValveSystem(SystemDef):
    """models/valve.hpp:64-103."""

    model_id = abi.MODEL_VALVE
    _dims = SystemDims(3, 5, 2, 2)

    def __init__(self, event_tolerance: float = 1e-6, ode: OdeControls | None = None):
        super().__init__(ode or OdeControls.uniform(3, 1e-10, 1e-10), (event_tolerance,))
        self.tol = event_tolerance

    def event_controls(self):
        return EventControls([-1, -1], [self.tol, self.tol], [1, 0], 50)


class DuffingLyapunovSystem(SystemDef):
    """models/duffing.hpp:162-180."""

    model_id = abi.MODEL_DUFFING_LYAPUNOV
    _dims = SystemDims(4, 4, 0, 1)

    def __init__(self, ode: OdeControls | None = None):
        super().__init__(ode or OdeControls.uniform(4, 1e-9, 1e-9))


# --------------------------------------------------------------- reference test fakes


def _one(rel=1e-9):
    return OdeControls.uniform(1, rel, rel)


class ConstantDef(SystemDef):
    """test_steppers.cpp:14-21."""

    model_id = abi.MODEL_CONSTANT
    _dims = SystemDims(1, 0, 0, 0)

    def __init__(self, value: float = 0.0):
        super().__init__(_one(), (value,))


class CubicTimeDef(SystemDef):
    """test_steppers.cpp:23-29."""

    model_id = abi.MODEL_CUBIC_TIME
    _dims = SystemDims(1, 0, 0, 0)

    def __init__(self):
        super().__init__(_one())


class ExponentialDef(SystemDef):
    """test_steppers.cpp:31-37."""

    model_id = abi.MODEL_EXPONENTIAL
    _dims = SystemDims(1, 0, 0, 0)

    def __init__(self):
        super().__init__(_one())


class UnitSlopeDef(SystemDef):
    """test_driver.cpp:17-23."""

    model_id = abi.MODEL_UNIT_SLOPE
    _dims = SystemDims(1, 0, 0, 0)

    def __init__(self):
        super().__init__(_one())


class BlowUpDef(SystemDef):
    """test_steppers.cpp:199-205."""

    model_id = abi.MODEL_BLOWUP
    _dims = SystemDims(1, 0, 0, 0)

    def __init__(self):
        super().__init__(_one())


class CountingDef(SystemDef):
    """test_driver.cpp:26-44."""

    model_id = abi.MODEL_COUNTING
    _dims = SystemDims(2, 4, 0, 3)

    def __init__(self):
        super().__init__(OdeControls.uniform(2, 1e-9, 1e-9))


class RampDef(SystemDef):
    """test_events.cpp:16-39."""

    model_id = abi.MODEL_RAMP
    _dims = SystemDims(1, 0, 1, 0)

    def __init__(self, slope=1.0, level=0.0, direction=0, stop=0, tol=1e-6, max_zone_steps=50):
        super().__init__(_one(), (slope, level, direction, stop, tol, max_zone_steps))
        self.direction, self.stop, self.tol, self.max_zone_steps = direction, stop, tol, max_zone_steps

    def event_controls(self):
        return EventControls([self.direction], [self.tol], [self.stop], self.max_zone_steps)


class DecayDef(SystemDef):
    """test_events.cpp:42-54."""

    model_id = abi.MODEL_DECAY
    _dims = SystemDims(1, 0, 1, 0)

    def __init__(self):
        super().__init__(_one())

    def event_controls(self):
        return EventControls([0], [1e-6], [0], 50)


class SeatContactDef(SystemDef):
    """test_events.cpp:56-68."""

    model_id = abi.MODEL_SEAT_CONTACT
    _dims = SystemDims(3, 5, 1, 0)

    def __init__(self):
        super().__init__(OdeControls.uniform(3, 1e-10, 1e-10))

    def event_controls(self):
        return EventControls([-1], [1e-6], [1])


class HarmonicDef(SystemDef):
    """test_driver.cpp:161-169."""

    model_id = abi.MODEL_HARMONIC
    _dims = SystemDims(2, 0, 0, 0)

    def __init__(self, ode: OdeControls | None = None):
        super().__init__(ode or OdeControls.uniform(2, 1e-6, 1e-6))
