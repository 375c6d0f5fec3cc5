// Pressure relief valve with impacts, hook side (device + host).
// Restates /root/reference/proj/include/odensemble/models/valve.hpp.
#ifndef ODEGPU_MODELS_VALVE_HPP
#define ODEGPU_MODELS_VALVE_HPP

#include <cmath>
#include <span>

#include "odegpu/hooks.hpp"

namespace odegpu::models {

/// valve.hpp:41-46; p = [kappa, delta, beta, q, r].
ODEGPU_HD ODEGPU_INLINE void valve_rhs(Real, std::span<const Real> y, std::span<const Real> p,
                                       std::span<Real> dy) {
    const Real kappa = p[0], delta = p[1], beta = p[2], q = p[3];
    dy[0] = y[1];
    dy[1] = -kappa * y[1] - (y[0] + delta) + y[2];
    dy[2] = beta * (q - y[0] * sqrt(y[2]));
}

/// Newtonian impact law on event 1 (y1 = 0 seat surface), valve.hpp:52-58.
ODEGPU_HD ODEGPU_INLINE void valve_impact_action(Index event_index, Real, std::span<Real> y,
                                                 std::span<const Real> p) {
    if (event_index == 1) {
        y[0] = 0.0;
        y[1] = -p[4] * y[1];
    }
}

/// ValveSystem (valve.hpp:64-103): F0 = y2 (stop at the next maximum),
/// F1 = y1 (impact action, continue); acc = running max/min of y1.
struct ValveHooks : HookDefaults {
    static constexpr Index kSystemDim = 3, kParamCount = 5, kEventCount = 2, kAccessoryCount = 2;
    ODEGPU_HD void ode_rhs(Real t, std::span<const Real> y, std::span<const Real> p, std::span<Real> dy) const {
        valve_rhs(t, y, p, dy);
    }
    ODEGPU_HD void event_values(Real, std::span<const Real> y, std::span<const Real>, std::span<Real> f) const {
        f[0] = y[1];
        f[1] = y[0];
    }
    ODEGPU_HD void event_action(Index event_index, Index, Real t, std::span<Real> y,
                                std::span<const Real> p) const {
        valve_impact_action(event_index, t, y, p);
    }
    ODEGPU_HD void initialize(Real, std::span<Real>, std::span<Real> y, std::span<const Real>,
                              std::span<Real> acc) const {
        acc[0] = y[0];
        acc[1] = y[0];
    }
    ODEGPU_HD void ordinary_accessory(Real, std::span<const Real> y, std::span<const Real>,
                                      std::span<Real> acc) const {
        // std::max / std::min semantics (valve.hpp:449-450)
        acc[0] = (acc[0] < y[0]) ? y[0] : acc[0];
        acc[1] = (y[0] < acc[1]) ? y[0] : acc[1];
    }
};

} // namespace odegpu::models

#endif
