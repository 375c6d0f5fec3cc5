// test_fakes.cuh — device restatements of the tiny SystemModels the
// reference's own test-suite defines (tests/test_steppers.cpp:14-45,
// tests/test_events.cpp:16-67, tests/test_driver.cpp:17-44, 161-169).
// Compiled into libodegpu so the reference's known-answer tests can be
// replayed through the product path (ODEGPU_MODEL_CONSTANT .. _BLOWUP).
#pragma once

#include <cmath>
#include <limits>
#include <span>

#include "odegpu/hooks.hpp"
#include "odegpu/models/duffing.hpp"
#include "odegpu/models/valve.hpp"

namespace odegpu::fakes {

struct OneDim : HookDefaults {
    static constexpr Index kSystemDim = 1, kParamCount = 0, kEventCount = 0, kAccessoryCount = 0;
};

struct ConstantHooks : OneDim { // y' = value
    Real value = 0;
    ODEGPU_HD void ode_rhs(Real, std::span<const Real>, std::span<const Real>, std::span<Real> dy) const {
        dy[0] = value;
    }
};

struct CubicTimeHooks : OneDim { // y' = t^3
    ODEGPU_HD void ode_rhs(Real t, std::span<const Real>, std::span<const Real>, std::span<Real> dy) const {
        dy[0] = t * t * t;
    }
};

struct ExponentialHooks : OneDim { // y' = y
    ODEGPU_HD void ode_rhs(Real, std::span<const Real> y, std::span<const Real>, std::span<Real> dy) const {
        dy[0] = y[0];
    }
};

struct UnitSlopeHooks : OneDim { // y' = 1
    ODEGPU_HD void ode_rhs(Real, std::span<const Real>, std::span<const Real>, std::span<Real> dy) const {
        dy[0] = 1.0;
    }
};

struct BlowUpHooks : OneDim { // y' = NaN
    ODEGPU_HD void ode_rhs(Real, std::span<const Real>, std::span<const Real>, std::span<Real> dy) const {
        dy[0] = std::numeric_limits<Real>::quiet_NaN();
    }
};

struct CountingHooks : HookDefaults { // duffing + hook call counters
    static constexpr Index kSystemDim = 2, kParamCount = 4, kEventCount = 0, kAccessoryCount = 3;
    ODEGPU_HD void ode_rhs(Real t, std::span<const Real> y, std::span<const Real> p, std::span<Real> dy) const {
        models::duffing_rhs(t, y, p, dy);
    }
    ODEGPU_HD void initialize(Real, std::span<Real>, std::span<Real>, std::span<const Real>,
                              std::span<Real> acc) const {
        acc[0] += 1;
    }
    ODEGPU_HD void finalize(Real, std::span<Real>, std::span<Real>, std::span<const Real>,
                            std::span<Real> acc) const {
        acc[1] += 1;
    }
    ODEGPU_HD void ordinary_accessory(Real, std::span<const Real>, std::span<const Real>,
                                      std::span<Real> acc) const {
        acc[2] += 1;
    }
};

struct RampHooks : HookDefaults { // y' = slope, F = y - level
    static constexpr Index kSystemDim = 1, kParamCount = 0, kEventCount = 1, kAccessoryCount = 0;
    Real slope = 1, level = 0;
    ODEGPU_HD void ode_rhs(Real, std::span<const Real>, std::span<const Real>, std::span<Real> dy) const {
        dy[0] = slope;
    }
    ODEGPU_HD void event_values(Real, std::span<const Real> y, std::span<const Real>, std::span<Real> f) const {
        f[0] = y[0] - level;
    }
};

struct DecayHooks : HookDefaults { // y' = -y, F = y
    static constexpr Index kSystemDim = 1, kParamCount = 0, kEventCount = 1, kAccessoryCount = 0;
    ODEGPU_HD void ode_rhs(Real, std::span<const Real> y, std::span<const Real>, std::span<Real> dy) const {
        dy[0] = -y[0];
    }
    ODEGPU_HD void event_values(Real, std::span<const Real> y, std::span<const Real>, std::span<Real> f) const {
        f[0] = y[0];
    }
};

struct SeatContactHooks : HookDefaults { // valve RHS, F = y1
    static constexpr Index kSystemDim = 3, kParamCount = 5, kEventCount = 1, kAccessoryCount = 0;
    ODEGPU_HD void ode_rhs(Real t, std::span<const Real> y, std::span<const Real> p, std::span<Real> dy) const {
        models::valve_rhs(t, y, p, dy);
    }
    ODEGPU_HD void event_values(Real, std::span<const Real> y, std::span<const Real>, std::span<Real> f) const {
        f[0] = y[0];
    }
};

struct HarmonicHooks : HookDefaults { // y1' = y2, y2' = -y1
    static constexpr Index kSystemDim = 2, kParamCount = 0, kEventCount = 0, kAccessoryCount = 0;
    ODEGPU_HD void ode_rhs(Real, std::span<const Real> y, std::span<const Real>, std::span<Real> dy) const {
        dy[0] = y[1];
        dy[1] = -y[0];
    }
};

} // namespace odegpu::fakes
