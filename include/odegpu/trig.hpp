// trig.hpp — libm functions for hook code, host and device.
//
// Hooks written against a Trig policy (template <class T> ... T::cos(x))
// compile for the host with <cmath> and for the solve kernels with
//   * the fast build: the libdevice-identical forms of
//     include/odegpu/device/dmath.cuh;
//   * the exact-parity build (make parity, ODEGPU_PARITY_BUILD): the
//     restatement of glibc 2.39's cos / sincos / pow in
//     include/odegpu/device/glibm.h — the libm the reference solver links,
//     bit for bit, so the device takes the reference's accept / reject and
//     event decisions exactly.
//
//   Trig           any argument; the range-reduction path for large |x|
//                  (libdevice's Payne-Hanek; in the parity build glibc's
//                  __branred range, |x| >= 105414350, which is not restated)
//                  sits behind one divergent branch per call.
//   CertifiedTrig  no range branch: straight-line code the scheduler can
//                  interleave across RK stages. Equal to Trig below
//                  kTrigCertifiedLimit and only ever run when the batch's trig
//                  certificate holds: a model that names `certified_hooks`
//                  (its hooks on CertifiedTrig) also provides
//                  trig_argument_bound(t0, t1, p, stride), a bound on
//                  |argument| of every trig call of a system integrated over
//                  [t0, t1]; a device pre-pass checks it for every system
//                  before each solve and the kernel picks the certified
//                  instantiation only if all pass (device/solver.cuh,
//                  trig_certificate_kernel).
#ifndef ODEGPU_TRIG_HPP
#define ODEGPU_TRIG_HPP

#include <cmath>

#include "odegpu/core.hpp"
#if defined(__CUDACC__)
#include "odegpu/device/dmath.cuh"
#include "odegpu/device/glibm.h"
#endif

#if defined(ODEGPU_PARITY_BUILD) && ODEGPU_PARITY_BUILD
#define ODEGPU_GLIBM 1
#else
#define ODEGPU_GLIBM 0
#endif

namespace odegpu {

struct Trig {
    ODEGPU_HD static ODEGPU_INLINE Real cos(Real x) {
#if defined(__CUDA_ARCH__) && ODEGPU_GLIBM
        return glm_trig_in_range(x) ? glm_cos(x) : device::dmath::cos(x);
#elif defined(__CUDA_ARCH__)
        return device::dmath::cos(x);
#else
        return std::cos(x);
#endif
    }
    ODEGPU_HD static ODEGPU_INLINE Real sin(Real x) {
#if defined(__CUDA_ARCH__) && ODEGPU_GLIBM
        Real s, c;
        if (!glm_trig_in_range(x)) return device::dmath::sin(x);
        glm_sincos(x, &s, &c);
        return s;
#elif defined(__CUDA_ARCH__)
        return device::dmath::sin(x);
#else
        return std::sin(x);
#endif
    }
    ODEGPU_HD static ODEGPU_INLINE void sincos(Real x, Real* s, Real* c) {
#if defined(__CUDA_ARCH__) && ODEGPU_GLIBM
        if (glm_trig_in_range(x)) glm_sincos(x, s, c);
        else device::dmath::sincos_fast(x, s, c);
#elif defined(__CUDA_ARCH__)
        device::dmath::sincos_fast(x, s, c);
#else
        *s = std::sin(x);
        *c = std::cos(x);
#endif
    }
};

struct CertifiedTrig {
    ODEGPU_HD static ODEGPU_INLINE Real cos(Real x) {
#if defined(__CUDA_ARCH__) && ODEGPU_GLIBM
        return glm_cos(x);
#elif defined(__CUDA_ARCH__)
        return device::dmath::cos_certified(x);
#else
        return std::cos(x);
#endif
    }
    ODEGPU_HD static ODEGPU_INLINE Real sin(Real x) {
#if defined(__CUDA_ARCH__) && ODEGPU_GLIBM
        Real s, c;
        glm_sincos(x, &s, &c);
        return s;
#elif defined(__CUDA_ARCH__)
        return device::dmath::sin_certified(x);
#else
        return std::sin(x);
#endif
    }
    ODEGPU_HD static ODEGPU_INLINE void sincos(Real x, Real* s, Real* c) {
#if defined(__CUDA_ARCH__) && ODEGPU_GLIBM
        glm_sincos(x, s, c);
#elif defined(__CUDA_ARCH__)
        device::dmath::sincos_certified(x, s, c);
#else
        *s = std::sin(x);
        *c = std::cos(x);
#endif
    }
};

/// std::pow of model code (the Keller-Miksis polytropic term): libdevice's
/// pow in the fast build, glibc's in the parity build, libm on the host.
ODEGPU_HD ODEGPU_INLINE Real libm_pow(Real x, Real y) {
#if defined(__CUDA_ARCH__) && ODEGPU_GLIBM
    return glm_pow(x, y);
#elif defined(__CUDA_ARCH__)
    return device::dmath::pow(x, y);
#else
    return std::pow(x, y);
#endif
}

/// Arguments strictly below this bound take the certified path: 2^31 (where
/// libdevice leaves its Cody-Waite reduction) or, in the parity build,
/// 105414350 (where glibc leaves reduce_sincos for __branred), less a
/// relative margin for the rounding of the argument's own arithmetic.
#if ODEGPU_GLIBM
inline constexpr Real kTrigCertifiedLimit = 105414350.0 * (1.0 - 1.0 / (1 << 20));
#else
inline constexpr Real kTrigCertifiedLimit = 2147483648.0 * (1.0 - 1.0 / (1 << 20));
#endif

} // namespace odegpu

#endif
