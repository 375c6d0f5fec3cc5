// Pressure relief valve with impacts, hook side (device + host).
// Restates /root/reference/proj/include/odensemble/models/valve.hpp.
#ifndef ODEGPU_MODELS_VALVE_HPP
#define ODEGPU_MODELS_VALVE_HPP

#include <cmath>
#include <span>
#include <stdexcept>

#include "odegpu/hooks.hpp"
#include "odegpu/system.hpp"

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
    static constexpr bool kTimeDomainUnchanged = true; // initialize writes accessories only
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

// ----------------------------------------------------------- host classes

/// Parameter slot order [kappa, delta, beta, q, r] (valve.hpp:17-37).
struct ValveParams {
    Real kappa = 1.25, delta = 10.0, beta = 20.0, q = 0.3, r = 0.8;
    static constexpr Index count = 5;
    void validate() const {
        if (!(r > 0 && r < 1)) throw std::invalid_argument("ValveParams: r must be in (0, 1)");
        if (!(q > 0)) throw std::invalid_argument("ValveParams: q must be > 0");
    }
    void write(std::span<Real> p) const {
        p[0] = kappa;
        p[1] = delta;
        p[2] = beta;
        p[3] = q;
        p[4] = r;
    }
};

/// valve.hpp:64-103
class ValveSystem : public ValveHooks {
public:
    using hooks_type = ValveHooks;
    explicit ValveSystem(Real event_tolerance = 1e-6, OdeControls ode = OdeControls::uniform(3, 1e-10, 1e-10))
        : tol_(event_tolerance), ode_(std::move(ode)) {}
    SystemDims dims() const { return dims_of<hooks_type>(); }
    OdeControls ode_controls() const { return ode_; }
    EventControls event_controls() const {
        return EventControls{.direction = {-1, -1}, .tolerance = {tol_, tol_}, .stop_condition = {1, 0},
                             .max_steps_in_zone = 50};
    }
    odegpu_model descriptor() const { return make_descriptor(ODEGPU_MODEL_VALVE, {tol_}); }

private:
    Real tol_;
    OdeControls ode_;
};

} // namespace odegpu::models

#endif
