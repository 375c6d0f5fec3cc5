// Duffing oscillator models, hook side (device + host).
// Restates /root/reference/proj/include/odensemble/models/duffing.hpp.
#ifndef ODEGPU_MODELS_DUFFING_HPP
#define ODEGPU_MODELS_DUFFING_HPP

#include <cmath>
#include <span>
#include <stdexcept>

#include "odegpu/hooks.hpp"
#include "odegpu/system.hpp"
#include "odegpu/trig.hpp"

namespace odegpu::models {

/// y1' = y2, y2' = delta*y1 - y1^3 - k*y2 + B*cos(omega*t); p = [k, B, delta, omega]
/// (duffing.hpp:37-42; same operation order).
template <class T = Trig>
ODEGPU_HD ODEGPU_INLINE void duffing_rhs(Real t, std::span<const Real> y, std::span<const Real> p,
                                         std::span<Real> dy) {
    const Real k = p[0], B = p[1], delta = p[2], omega = p[3];
    dy[0] = y[1];
    dy[1] = delta * y[0] - y[0] * y[0] * y[0] - k * y[1] + B * T::cos(omega * t);
}

/// Duffing + linearised radius/angle (duffing.hpp:47-57).
ODEGPU_HD ODEGPU_INLINE void duffing_lyapunov_rhs(Real t, std::span<const Real> y, std::span<const Real> p,
                                                  std::span<Real> dy) {
    duffing_rhs<Trig>(t, y, p, dy);
    const Real k = p[0], delta = p[2];
    const Real g1 = delta - 3.0 * y[0] * y[0];
    const Real g2 = -k;
    Real s, c;
    Trig::sincos(y[3], &s, &c); // state-dependent argument: never certified
    dy[2] = y[2] * ((1.0 + g1) * s * c + g2 * s * s);
    dy[3] = -s * s + (g1 * c + g2 * s) * c;
}

/// DuffingSystem (duffing.hpp:75-88): plain RHS. The only trig argument is
/// omega*t, so |argument| <= |omega| max(|t0|, |t1|) certifies a system.
template <class T = Trig>
struct DuffingHooksT : HookDefaults {
    static constexpr Index kSystemDim = 2, kParamCount = 4, kEventCount = 0, kAccessoryCount = 0;
    ODEGPU_HD void ode_rhs(Real t, std::span<const Real> y, std::span<const Real> p, std::span<Real> dy) const {
        duffing_rhs<T>(t, y, p, dy);
    }
    // time split (hooks.hpp TimeSplitHooks): the forcing cos(omega t)
    static constexpr Index kTimeTermCount = 1;
    ODEGPU_HD void time_terms(Real t, std::span<const Real> p, std::span<Real> tt) const {
        tt[0] = T::cos(p[3] * t);
    }
    ODEGPU_HD void ode_rhs_split(Real, std::span<const Real> y, std::span<const Real> p, std::span<const Real> tt,
                                 std::span<Real> dy) const {
        const Real k = p[0], B = p[1], delta = p[2];
        dy[0] = y[1];
        dy[1] = delta * y[0] - y[0] * y[0] * y[0] - k * y[1] + B * tt[0];
    }
    ODEGPU_HD static Real trig_argument_bound(Real t0, Real t1, const Real* p, Index stride) {
        return fabs(p[3 * stride]) * fmax(fabs(t0), fabs(t1));
    }
};

/// DuffingMaxAccessorySystem (duffing.hpp:92-117): running max of y1 + time.
template <class T = Trig>
struct DuffingMaxAccessoryHooksT : DuffingHooksT<T> {
    static constexpr bool kTimeDomainUnchanged = true; // initialize writes state / accessories only
    static constexpr Index kAccessoryCount = 2;
    using certified_hooks = DuffingMaxAccessoryHooksT<CertifiedTrig>;
    ODEGPU_HD void initialize(Real t, std::span<Real>, std::span<Real> y, std::span<const Real>,
                              std::span<Real> acc) const {
        acc[0] = y[0];
        acc[1] = t;
    }
    ODEGPU_HD void ordinary_accessory(Real t, std::span<const Real> y, std::span<const Real>,
                                      std::span<Real> acc) const {
        if (y[0] > acc[0]) {
            acc[0] = y[0];
            acc[1] = t;
        }
    }
};

/// DuffingMaxEventSystem (duffing.hpp:122-156): F = y2 falling locates the
/// local maxima of y1; the event accessory keeps the largest and its time.
template <class T = Trig>
struct DuffingMaxEventHooksT : DuffingHooksT<T> {
    static constexpr bool kTimeDomainUnchanged = true; // initialize writes state / accessories only
    static constexpr Index kEventCount = 1, kAccessoryCount = 2;
    using certified_hooks = DuffingMaxEventHooksT<CertifiedTrig>;
    ODEGPU_HD void event_values(Real, std::span<const Real> y, std::span<const Real>, std::span<Real> f) const {
        f[0] = y[1];
    }
    ODEGPU_HD void initialize(Real t, std::span<Real>, std::span<Real> y, std::span<const Real>,
                              std::span<Real> acc) const {
        acc[0] = y[0];
        acc[1] = t;
    }
    ODEGPU_HD void event_accessory(Index event, Index, Real t, std::span<const Real> y, std::span<const Real>,
                                   std::span<Real> acc) const {
        if (event == 0 && y[0] > acc[0]) {
            acc[0] = y[0];
            acc[1] = t;
        }
    }
};

/// cfg1 harness model: per-period max and min of y1 with
/// their times, acc = [y1_max, t_max, y1_min, t_min], seeded at t0.
template <class T = Trig>
struct DuffingMaxMinHooksT : DuffingHooksT<T> {
    static constexpr bool kTimeDomainUnchanged = true; // initialize writes state / accessories only
    static constexpr Index kAccessoryCount = 4;
    using certified_hooks = DuffingMaxMinHooksT<CertifiedTrig>;
    ODEGPU_HD void initialize(Real t, std::span<Real>, std::span<Real> y, std::span<const Real>,
                              std::span<Real> acc) const {
        acc[0] = y[0];
        acc[1] = t;
        acc[2] = y[0];
        acc[3] = t;
    }
    ODEGPU_HD void ordinary_accessory(Real t, std::span<const Real> y, std::span<const Real>,
                                      std::span<Real> acc) const {
        if (y[0] > acc[0]) {
            acc[0] = y[0];
            acc[1] = t;
        }
        if (y[0] < acc[2]) {
            acc[2] = y[0];
            acc[3] = t;
        }
    }
};

/// Plain Duffing with the certified path.
struct DuffingHooks : DuffingHooksT<Trig> {
    using certified_hooks = DuffingHooksT<CertifiedTrig>;
};
using DuffingMaxAccessoryHooks = DuffingMaxAccessoryHooksT<Trig>;
using DuffingMaxEventHooks = DuffingMaxEventHooksT<Trig>;
using DuffingMaxMinHooks = DuffingMaxMinHooksT<Trig>;

/// DuffingLyapunovSystem (duffing.hpp:162-180): finalize samples the
/// linearised radius into acc[0] and resets it to one.
struct DuffingLyapunovHooks : HookDefaults {
    static constexpr Index kSystemDim = 4, kParamCount = 4, kEventCount = 0, kAccessoryCount = 1;
    ODEGPU_HD void ode_rhs(Real t, std::span<const Real> y, std::span<const Real> p, std::span<Real> dy) const {
        duffing_lyapunov_rhs(t, y, p, dy);
    }
    ODEGPU_HD void finalize(Real, std::span<Real>, std::span<Real> y, std::span<const Real>,
                            std::span<Real> acc) const {
        acc[0] = y[2];
        y[2] = 1.0;
    }
    static constexpr bool kFinalizeKeepsTimeDomain = true; // finalize never writes td (hooks.hpp)
    static constexpr bool kTimeDomainUnchanged = true;
};

// ----------------------------------------------------------- host classes
// Same names, constructors and controls as the reference
// (duffing.hpp:17-35, 75-180); hooks come from the *Hooks bases above.

/// Parameter slot order [k, B, delta, omega] (duffing.hpp:17-35).
struct DuffingParams {
    Real k = 0.2, B = 0.3, delta = 1.0, omega = 1.0;
    static constexpr Index count = 4;
    void validate() const {
        if (!(B > 0) || !(omega > 0)) throw std::invalid_argument("DuffingParams: B and omega must be > 0");
    }
    void write(std::span<Real> p) const {
        p[0] = k;
        p[1] = B;
        p[2] = delta;
        p[3] = omega;
    }
};

template <class H, int ID>
class DuffingFamily : public H {
public:
    using hooks_type = H;
    explicit DuffingFamily(OdeControls ode = OdeControls::uniform(H::kSystemDim, 1e-9, 1e-9))
        : ode_(std::move(ode)) {}
    SystemDims dims() const { return dims_of<H>(); }
    OdeControls ode_controls() const { return ode_; }
    EventControls event_controls() const { return {}; }
    odegpu_model descriptor() const { return make_descriptor(ID); }

private:
    OdeControls ode_;
};

using DuffingSystem = DuffingFamily<DuffingHooks, ODEGPU_MODEL_DUFFING>;
using DuffingMaxAccessorySystem = DuffingFamily<DuffingMaxAccessoryHooks, ODEGPU_MODEL_DUFFING_MAX_ACCESSORY>;
using DuffingMaxMinSystem = DuffingFamily<DuffingMaxMinHooks, ODEGPU_MODEL_DUFFING_MAXMIN>;
using DuffingLyapunovSystem = DuffingFamily<DuffingLyapunovHooks, ODEGPU_MODEL_DUFFING_LYAPUNOV>;

/// duffing.hpp:122-156
class DuffingMaxEventSystem : public DuffingMaxEventHooks {
public:
    using hooks_type = DuffingMaxEventHooks;
    explicit DuffingMaxEventSystem(Real event_tolerance = 1e-6, Index stop_after = 0,
                                   OdeControls ode = OdeControls::uniform(2, 1e-9, 1e-9))
        : tol_(event_tolerance), stop_(stop_after), ode_(std::move(ode)) {}
    SystemDims dims() const { return dims_of<hooks_type>(); }
    OdeControls ode_controls() const { return ode_; }
    EventControls event_controls() const {
        return EventControls{.direction = {-1}, .tolerance = {tol_}, .stop_condition = {stop_}};
    }
    odegpu_model descriptor() const {
        return make_descriptor(ODEGPU_MODEL_DUFFING_MAX_EVENT, {tol_, static_cast<double>(stop_)});
    }

private:
    Real tol_;
    Index stop_;
    OdeControls ode_;
};

/// duffing.hpp:62-71: lambda = sum(ln sample_n) / (N * period).
inline Real lyapunov_accumulate(std::span<const Real> samples, Real period) {
    if (samples.empty()) throw std::invalid_argument("lyapunov_accumulate: no samples");
    if (!(period > 0)) throw std::invalid_argument("lyapunov_accumulate: period must be > 0");
    Real sum = 0;
    for (Real s : samples) {
        if (!(s > 0)) throw std::invalid_argument("lyapunov_accumulate: nonpositive sample");
        sum += std::log(s);
    }
    return sum / (static_cast<Real>(std::ssize(samples)) * period);
}

} // namespace odegpu::models

#endif
