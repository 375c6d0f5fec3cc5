// trig.hpp — trigonometry for hook code, host and device.
//
// Hooks written against a Trig policy (template <class T> ... T::cos(x))
// compile for the host with <cmath> and for the solve kernels with the
// libdevice-identical forms of include/odegpu/device/dmath.cuh:
//
//   Trig           any argument; libdevice's Payne-Hanek path for |x| >= 2^31
//                  sits behind one divergent branch per call.
//   CertifiedTrig  no range branch: straight-line code the scheduler can
//                  interleave across RK stages. Equal to Trig for |x| < 2^31
//                  and only ever run when the batch's trig certificate holds:
//                  a model that names `certified_hooks` (its hooks on
//                  CertifiedTrig) also provides trig_argument_bound(t0, t1,
//                  p, stride), a bound on |argument| of every trig call of a
//                  system integrated over [t0, t1]; a device pre-pass checks
//                  it for every system before each solve and the kernel picks
//                  the certified instantiation only if all pass
//                  (device/solver.cuh, trig_certificate_kernel).
#ifndef ODEGPU_TRIG_HPP
#define ODEGPU_TRIG_HPP

#include <cmath>

#include "odegpu/core.hpp"
#if defined(__CUDACC__)
#include "odegpu/device/dmath.cuh"
#endif

namespace odegpu {

struct Trig {
    ODEGPU_HD static ODEGPU_INLINE Real cos(Real x) {
#if defined(__CUDA_ARCH__)
        return device::dmath::cos(x);
#else
        return std::cos(x);
#endif
    }
    ODEGPU_HD static ODEGPU_INLINE Real sin(Real x) {
#if defined(__CUDA_ARCH__)
        return device::dmath::sin(x);
#else
        return std::sin(x);
#endif
    }
    ODEGPU_HD static ODEGPU_INLINE void sincos(Real x, Real* s, Real* c) {
#if defined(__CUDA_ARCH__)
        device::dmath::sincos_fast(x, s, c);
#else
        *s = std::sin(x);
        *c = std::cos(x);
#endif
    }
};

struct CertifiedTrig {
    ODEGPU_HD static ODEGPU_INLINE Real cos(Real x) {
#if defined(__CUDA_ARCH__)
        return device::dmath::cos_certified(x);
#else
        return std::cos(x);
#endif
    }
    ODEGPU_HD static ODEGPU_INLINE Real sin(Real x) {
#if defined(__CUDA_ARCH__)
        return device::dmath::sin_certified(x);
#else
        return std::sin(x);
#endif
    }
    ODEGPU_HD static ODEGPU_INLINE void sincos(Real x, Real* s, Real* c) {
#if defined(__CUDA_ARCH__)
        device::dmath::sincos_certified(x, s, c);
#else
        *s = std::sin(x);
        *c = std::cos(x);
#endif
    }
};

/// Arguments strictly below this bound take the certified path (2^31 less a
/// relative margin for the rounding of the argument's own arithmetic).
inline constexpr Real kTrigCertifiedLimit = 2147483648.0 * (1.0 - 1.0 / (1 << 20));

} // namespace odegpu

#endif
