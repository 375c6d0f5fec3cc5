// Keller-Miksis bubble models, hook side (device + host).
// Restates /root/reference/proj/include/odensemble/models/keller_miksis.hpp.
// The 13 coefficients are precomputed on the host (bubble_coefficients,
// keller_miksis.hpp:47-77; see paper_1810_03931_b200/workloads.py and
// include/odegpu/system.hpp) and are per-system parameters.
#ifndef ODEGPU_MODELS_KELLER_MIKSIS_HPP
#define ODEGPU_MODELS_KELLER_MIKSIS_HPP

#include <cmath>
#include <limits>
#include <span>
#include <stdexcept>

#include "odegpu/hooks.hpp"
#include "odegpu/system.hpp"
#include "odegpu/trig.hpp"

namespace odegpu::models {

/// The excitation terms of the Keller-Miksis RHS, which depend on tau and
/// the coefficients only: tt = [c5 sin(2 pi tau) + c6 sin(arg2),
/// c7 cos(2 pi tau) + c8 cos(arg2)], arg2 = 2 pi c11 tau + c12
/// (keller_miksis.hpp:93-99). On the device sin/cos of the same argument
/// share one range reduction (sincos), as the reference's g++ build merges
/// them into glibc sincos.
template <class T = Trig>
ODEGPU_HD ODEGPU_INLINE void keller_miksis_time_terms(Real tau, std::span<const Real> c, std::span<Real> tt) {
    constexpr Real two_pi = 2.0 * 3.141592653589793238462643383279502884;
    const Real arg1 = two_pi * tau;
    const Real arg2 = two_pi * c[11] * tau + c[12];
    Real s1, c1, s2, c2;
    T::sincos(arg1, &s1, &c1);
    // single-frequency excitation (f2 = f1, theta = 0: the scans' and
    // BASELINE's bubble pools) gives arg2 == arg1 bit for bit, and sincos is
    // a function of its argument: reuse the values instead of recomputing
    // them (bitwise the same terms; the reference evaluates both)
    if (arg2 == arg1) {
        s2 = s1;
        c2 = c1;
    } else {
        T::sincos(arg2, &s2, &c2);
    }
    tt[0] = c[5] * s1 + c[6] * s2;
    tt[1] = c[7] * c1 + c[8] * c2;
}

/// Dimensionless Keller-Miksis RHS (keller_miksis.hpp:82-103) given its
/// excitation terms, same operation order. y1 <= 0 yields NaN derivatives
/// for the step control.
ODEGPU_HD ODEGPU_INLINE void keller_miksis_rhs_split(std::span<const Real> y, std::span<const Real> c,
                                                     std::span<const Real> tt, std::span<Real> dy) {
    const Real y1 = y[0], y2 = y[1];
    if (!(y1 > 0)) {
        dy[0] = std::numeric_limits<Real>::quiet_NaN();
        dy[1] = std::numeric_limits<Real>::quiet_NaN();
        return;
    }
#if defined(__CUDA_ARCH__) && !ODEGPU_GLIBM
    // Every quotient of the RHS through the division fast path without its
    // per-division branch (1/y1, c3/y1 and c4 y2/y1 share one reciprocal of
    // y1; /3 uses RN(1/3)) and pow in its branch-free form — bitwise the
    // same values (dmath.cuh: Divisor, pow_lean). The RHS is straight-line
    // code the scheduler can interleave; two rarely taken branches redo the
    // quotients the general way when an operand leaves the fast forms' range.
    device::dmath::Divisor by_y1(y1);
    device::dmath::Divisor by_3(3.0, 1.0 / 3.0);
    Real inv = by_y1.reciprocal();
    Real q3 = by_y1.div(c[3]);
    Real q4 = by_y1.div(c[4] * y2);
    Real third = by_3.div(c[9] * y2);
    bool lean = true;
    Real pw = device::dmath::pow_lean(inv, c[10], &lean);
    if (!(by_y1.ok() && by_3.ok() && lean)) {
        inv = 1.0 / y1;
        q3 = c[3] / y1;
        q4 = c[4] * y2 / y1;
        third = c[9] * y2 / 3.0;
        pw = device::dmath::pow(inv, c[10]);
    }
    const Real numerator = (c[0] + c[1] * y2) * pw - c[2] * (1.0 + c[9] * y2) - q3 - q4 -
                           (1.0 - third) * 1.5 * y2 * y2 - tt[0] * (1.0 + c[9] * y2) - y1 * tt[1];
    const Real denominator = y1 - c[9] * y1 * y2 + c[4] * c[9];
    device::dmath::Divisor by_den(denominator);
    Real ddy = by_den.div(numerator);
    if (!by_den.ok()) ddy = numerator / denominator;
    dy[0] = y2;
    dy[1] = ddy;
#else
    // host, and the exact-parity build: the reference's expression with its
    // libm's pow (glibc restated on the device, include/odegpu/device/glibm.h)
    const Real pw = libm_pow(1.0 / y1, c[10]);
    const Real numerator = (c[0] + c[1] * y2) * pw - c[2] * (1.0 + c[9] * y2) - c[3] / y1 - c[4] * y2 / y1 -
                           (1.0 - c[9] * y2 / 3.0) * 1.5 * y2 * y2 - tt[0] * (1.0 + c[9] * y2) - y1 * tt[1];
    const Real denominator = y1 - c[9] * y1 * y2 + c[4] * c[9];
    dy[0] = y2;
    dy[1] = numerator / denominator;
#endif
}

/// Dimensionless Keller-Miksis RHS (keller_miksis.hpp:82-103).
template <class T = Trig>
ODEGPU_HD ODEGPU_INLINE void keller_miksis_rhs(Real tau, std::span<const Real> y, std::span<const Real> c,
                                               std::span<Real> dy) {
    Real tt[2];
    keller_miksis_time_terms<T>(tau, c, std::span<Real>(tt, 2));
    keller_miksis_rhs_split(y, c, std::span<const Real>(tt, 2), dy);
}

/// KellerMiksisSystem (keller_miksis.hpp:106-119). Trig arguments 2 pi tau and
/// 2 pi c11 tau + c12: |argument| <= 2 pi max|tau| max(1, |c11|) + |c12|.
template <class T = Trig>
struct KellerMiksisHooksT : HookDefaults {
    static constexpr Index kSystemDim = 2, kParamCount = 13, kEventCount = 0, kAccessoryCount = 0;
    using certified_hooks = KellerMiksisHooksT<CertifiedTrig>;
    ODEGPU_HD void ode_rhs(Real t, std::span<const Real> y, std::span<const Real> p, std::span<Real> dy) const {
        keller_miksis_rhs<T>(t, y, p, dy);
    }
    // time split (hooks.hpp TimeSplitHooks): the two excitation terms
    static constexpr Index kTimeTermCount = 2;
    ODEGPU_HD void time_terms(Real t, std::span<const Real> p, std::span<Real> tt) const {
        keller_miksis_time_terms<T>(t, p, tt);
    }
    ODEGPU_HD void ode_rhs_split(Real, std::span<const Real> y, std::span<const Real> p, std::span<const Real> tt,
                                 std::span<Real> dy) const {
        keller_miksis_rhs_split(y, p, tt, dy);
    }
    ODEGPU_HD static Real trig_argument_bound(Real t0, Real t1, const Real* p, Index stride) {
        constexpr Real two_pi = 2.0 * 3.141592653589793238462643383279502884;
        return two_pi * fmax(fabs(t0), fabs(t1)) * fmax(1.0, fabs(p[11 * stride])) + fabs(p[12 * stride]);
    }
};

/// BubbleCollapseSystem (keller_miksis.hpp:126-165): runs from one radius
/// maximum to the next (F = y2 falling, stop at 1); acc = [tau_max, y1_max,
/// tau_min, y1_min]; finalize moves t0 to the stop time.
template <class T = Trig>
struct BubbleCollapseHooksT : KellerMiksisHooksT<T> {
    static constexpr Index kEventCount = 1, kAccessoryCount = 4;
    using certified_hooks = BubbleCollapseHooksT<CertifiedTrig>;
    ODEGPU_HD void event_values(Real, std::span<const Real> y, std::span<const Real>, std::span<Real> f) const {
        f[0] = y[1];
    }
    ODEGPU_HD void initialize(Real t, std::span<Real>, std::span<Real> y, std::span<const Real>,
                              std::span<Real> acc) const {
        acc[0] = t;
        acc[1] = y[0];
        acc[2] = t;
        acc[3] = y[0];
    }
    ODEGPU_HD void ordinary_accessory(Real t, std::span<const Real> y, std::span<const Real>,
                                      std::span<Real> acc) const {
        if (y[0] < acc[3]) {
            acc[3] = y[0];
            acc[2] = t;
        }
    }
    ODEGPU_HD void finalize(Real t, std::span<Real> time_domain, std::span<Real>, std::span<const Real>,
                            std::span<Real>) const {
        time_domain[0] = t;
    }
    // finalize moves t0 to the stop time t in [t0, t1] (hooks.hpp)
    static constexpr bool kFinalizeKeepsTimeDomain = true;
};

using KellerMiksisHooks = KellerMiksisHooksT<Trig>;
using BubbleCollapseHooks = BubbleCollapseHooksT<Trig>;

// ----------------------------------------------------------- host classes

/// Physical description of a dual-frequency driven bubble; defaults are
/// water with a 10 micron bubble (keller_miksis.hpp:18-32).
struct BubblePhysical {
    Real pa1 = 0, pa2 = 0, omega1 = 0, omega2 = 0, theta = 0;
    Real R_E = 10e-6, c_L = 1497.3, rho_L = 997.1, P_inf = 1.0e5, p_V = 3166.8, sigma = 0.072,
         mu_L = 8.902e-4, gamma = 1.4;
};

/// The 13 dimensionless coefficients (keller_miksis.hpp:36-45).
struct BubbleCoefficients {
    Real c[13]{};
    static constexpr Index count = 13;
    Real operator[](std::size_t i) const { return c[i]; }
    void write(std::span<Real> p) const {
        for (std::size_t i = 0; i < 13; ++i) p[i] = c[i];
    }
};

/// keller_miksis.hpp:47-77, same operation order (bitwise equal results).
inline BubbleCoefficients bubble_coefficients(const BubblePhysical& phys) {
    if (!(phys.omega1 > 0)) throw std::invalid_argument("bubble_coefficients: omega1 must be > 0");
    if (!(phys.R_E > 0)) throw std::invalid_argument("bubble_coefficients: R_E must be > 0");
    if (!(phys.gamma > 1)) throw std::invalid_argument("bubble_coefficients: gamma must be > 1");
    if (!(phys.rho_L > 0) || !(phys.c_L > 0))
        throw std::invalid_argument("bubble_coefficients: invalid material constants");
    constexpr Real two_pi = 2.0 * 3.141592653589793238462643383279502884;
    const Real w = phys.R_E * phys.omega1;
    const Real S = two_pi / w;
    const Real G = S * S / phys.rho_L;
    const Real A = phys.P_inf - phys.p_V;
    const Real B = 2.0 * phys.sigma / phys.R_E;
    BubbleCoefficients out;
    Real* c = out.c;
    c[0] = (A + B) * G;
    c[1] = (1.0 - 3.0 * phys.gamma) * (A + B) * S / (phys.rho_L * phys.c_L);
    c[2] = A * G;
    c[3] = B * G;
    c[4] = 4.0 * phys.mu_L / (phys.rho_L * phys.R_E * phys.R_E) * (two_pi / phys.omega1);
    c[5] = phys.pa1 * G;
    c[6] = phys.pa2 * G;
    c[7] = (w / phys.c_L) * c[5];
    c[8] = (w / phys.c_L) * c[6];
    c[9] = w / (two_pi * phys.c_L);
    c[10] = 3.0 * phys.gamma;
    c[11] = phys.omega2 / phys.omega1;
    c[12] = phys.theta;
    return out;
}

/// keller_miksis.hpp:106-119
class KellerMiksisSystem : public KellerMiksisHooks {
public:
    using hooks_type = KellerMiksisHooks;
    explicit KellerMiksisSystem(OdeControls ode = OdeControls::uniform(2, 1e-10, 1e-10)) : ode_(std::move(ode)) {}
    SystemDims dims() const { return dims_of<hooks_type>(); }
    OdeControls ode_controls() const { return ode_; }
    EventControls event_controls() const { return {}; }
    odegpu_model descriptor() const { return make_descriptor(ODEGPU_MODEL_KELLER_MIKSIS); }

private:
    OdeControls ode_;
};

/// keller_miksis.hpp:126-165
class BubbleCollapseSystem : public BubbleCollapseHooks {
public:
    using hooks_type = BubbleCollapseHooks;
    explicit BubbleCollapseSystem(Real event_tolerance = 1e-6,
                                  OdeControls ode = OdeControls::uniform(2, 1e-10, 1e-10))
        : tol_(event_tolerance), ode_(std::move(ode)) {}
    SystemDims dims() const { return dims_of<hooks_type>(); }
    OdeControls ode_controls() const { return ode_; }
    EventControls event_controls() const {
        return EventControls{.direction = {-1}, .tolerance = {tol_}, .stop_condition = {1}};
    }
    odegpu_model descriptor() const { return make_descriptor(ODEGPU_MODEL_BUBBLE_COLLAPSE, {tol_}); }

private:
    Real tol_;
    OdeControls ode_;
};

} // namespace odegpu::models

#endif
