// solver.cuh — the sm_100a ensemble kernel: one thread integrates one system
// at a time, entirely in registers; a lane that finishes its system fetches
// the next one from a global work counter (warp-aggregated atomics), so warps
// stay full until the pool drains.
//
// Semantics are exactly those of the reference's per-system loop
// (/root/reference/proj/include/odensemble/driver.hpp:83-234) with the
// RK4 / Cash-Karp steppers (steppers.hpp:82-139), error control
// (steppers.hpp:154-198), event machine (events.hpp:22-178) and secant
// location (events.hpp:200-241). The loop is restructured as a per-lane
// state machine so that *every* Runge-Kutta evaluation — a normal trial
// step or a secant re-step — goes through one shared call site: lanes in
// different phases (stepping, locating an event, committing, refilling)
// still execute the expensive RK stages together. Divergence is confined
// to the cheap bookkeeping between steps.
#ifndef ODEGPU_DEVICE_SOLVER_CUH
#define ODEGPU_DEVICE_SOLVER_CUH

#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <span>

#include "odegpu/hooks.hpp"

namespace odegpu::device {

constexpr int kMaxDim = 8;
constexpr int kMaxEvents = 4;

/// Shared read-only controls, materialised once per solve (solve.hpp:153-155)
/// and passed in the kernel parameter bank (constant cache).
struct Controls {
    Real rel_tol[kMaxDim];
    Real abs_tol[kMaxDim];
    Real max_step, min_step, step_grow_limit, step_shrink_limit;
    Real initial_time_step;
    Real tolerance[kMaxEvents];
    Index stop_condition[kMaxEvents];
    int direction[kMaxEvents];
    Index max_steps_in_zone;
};

/// Device SoA arrays of one batch (stride n): batch.hpp:61-66, outcomes
/// split per field so every store is coalesced.
struct BatchArrays {
    Real* td;        // [2n]
    Real* state;     // [dim n]
    const Real* params;
    Real* acc;
    Real* final_t;
    std::uint8_t* reason;
    Index* accepted;
    Index* rejected;
    Index* detections;
    Index* secant_failures;
    Real* smallest_step;
    Index n;
    unsigned long long* work; // next system to hand out (zeroed before launch)
};

// --- Cash-Karp tableau (steppers.hpp:16-39): exact rationals rendered once.
namespace ck {
constexpr Real c2 = 1.0 / 5.0, c3 = 3.0 / 10.0, c4 = 3.0 / 5.0, c5 = 1.0, c6 = 7.0 / 8.0;
constexpr Real a21 = 1.0 / 5.0;
constexpr Real a31 = 3.0 / 40.0, a32 = 9.0 / 40.0;
constexpr Real a41 = 3.0 / 10.0, a42 = -9.0 / 10.0, a43 = 6.0 / 5.0;
constexpr Real a51 = -11.0 / 54.0, a52 = 5.0 / 2.0, a53 = -70.0 / 27.0, a54 = 35.0 / 27.0;
constexpr Real a61 = 1631.0 / 55296.0, a62 = 175.0 / 512.0, a63 = 575.0 / 13824.0, a64 = 44275.0 / 110592.0,
               a65 = 253.0 / 4096.0;
constexpr Real b1 = 37.0 / 378.0, b3 = 250.0 / 621.0, b4 = 125.0 / 594.0, b6 = 512.0 / 1771.0;
constexpr Real e1 = 2825.0 / 27648.0, e3 = 18575.0 / 48384.0, e4 = 13525.0 / 55296.0, e5 = 277.0 / 14336.0,
               e6 = 1.0 / 4.0;
constexpr Real d1 = b1 - e1, d3 = b3 - e3, d4 = b4 - e4, d5 = -e5, d6 = b6 - e6;
} // namespace ck

// std::max / std::min / std::clamp semantics, including NaN behaviour.
__device__ __forceinline__ Real smax(Real a, Real b) { return (a < b) ? b : a; }
__device__ __forceinline__ Real smin(Real a, Real b) { return (b < a) ? b : a; }
__device__ __forceinline__ Real sclamp(Real v, Real lo, Real hi) { return (v < lo) ? lo : (hi < v) ? hi : v; }

template <int N>
using Vec = Real[N];

template <class H>
__device__ __forceinline__ void rhs(const H& m, Real t, const Real (&y)[H::kSystemDim],
                                    const Real* p, Real (&dy)[H::kSystemDim]) {
    m.ode_rhs(t, std::span<const Real>(y, H::kSystemDim), std::span<const Real>(p, H::kParamCount),
              std::span<Real>(dy, H::kSystemDim));
}

/// One trial step from (t, y) with step h (steppers.hpp:82-139). Writes the
/// proposed state, the embedded error |y5 - y4| (RKCK45) and whether
/// anything is non-finite.
template <class H, Algorithm ALG>
__device__ __forceinline__ bool rk_step(const H& m, Real t, Real h, const Real (&y)[H::kSystemDim],
                                        const Real* p, Real (&out)[H::kSystemDim],
                                        Real (&err)[H::kSystemDim]) {
    constexpr int N = H::kSystemDim;
    Real k1[N], k2[N], k3[N], k4[N], yt[N];
    bool finite = true;
    if constexpr (ALG == Algorithm::RK4) {
        rhs(m, t, y, p, k1);
#pragma unroll
        for (int i = 0; i < N; ++i) yt[i] = y[i] + 0.5 * h * k1[i];
        rhs(m, t + 0.5 * h, yt, p, k2);
#pragma unroll
        for (int i = 0; i < N; ++i) yt[i] = y[i] + 0.5 * h * k2[i];
        rhs(m, t + 0.5 * h, yt, p, k3);
#pragma unroll
        for (int i = 0; i < N; ++i) yt[i] = y[i] + h * k3[i];
        rhs(m, t + h, yt, p, k4);
#pragma unroll
        for (int i = 0; i < N; ++i) {
            out[i] = y[i] + (h / 6.0) * (k1[i] + 2.0 * k2[i] + 2.0 * k3[i] + k4[i]);
            err[i] = 0.0;
            finite = finite && isfinite(out[i]);
        }
    } else {
        Real k5[N], k6[N];
        rhs(m, t, y, p, k1);
#pragma unroll
        for (int i = 0; i < N; ++i) yt[i] = y[i] + h * (ck::a21 * k1[i]);
        rhs(m, t + ck::c2 * h, yt, p, k2);
#pragma unroll
        for (int i = 0; i < N; ++i) yt[i] = y[i] + h * (ck::a31 * k1[i] + ck::a32 * k2[i]);
        rhs(m, t + ck::c3 * h, yt, p, k3);
#pragma unroll
        for (int i = 0; i < N; ++i) yt[i] = y[i] + h * (ck::a41 * k1[i] + ck::a42 * k2[i] + ck::a43 * k3[i]);
        rhs(m, t + ck::c4 * h, yt, p, k4);
#pragma unroll
        for (int i = 0; i < N; ++i)
            yt[i] = y[i] + h * (ck::a51 * k1[i] + ck::a52 * k2[i] + ck::a53 * k3[i] + ck::a54 * k4[i]);
        rhs(m, t + ck::c5 * h, yt, p, k5);
#pragma unroll
        for (int i = 0; i < N; ++i)
            yt[i] = y[i] + h * (ck::a61 * k1[i] + ck::a62 * k2[i] + ck::a63 * k3[i] + ck::a64 * k4[i] +
                                ck::a65 * k5[i]);
        rhs(m, t + ck::c6 * h, yt, p, k6);
#pragma unroll
        for (int i = 0; i < N; ++i) {
            out[i] = y[i] + h * (ck::b1 * k1[i] + ck::b3 * k3[i] + ck::b4 * k4[i] + ck::b6 * k6[i]);
            err[i] = fabs(h * (ck::d1 * k1[i] + ck::d3 * k3[i] + ck::d4 * k4[i] + ck::d5 * k5[i] + ck::d6 * k6[i]));
            finite = finite && isfinite(out[i]) && isfinite(err[i]);
        }
    }
    return !finite;
}

// Event zones (events.hpp:22-26) and transitions (events.hpp:54-70).
enum : int { kZoneNone = -1, kZoneBelow = 0, kZoneInside = 1, kZoneAbove = 2 };
enum : int { kKindNone = -1, kKindAcross = 0, kKindEntered = 1 };

__device__ __forceinline__ int zone_of(Real v, Real tol) {
    if (!isfinite(v)) return kZoneNone;
    if (fabs(v) <= tol) return kZoneInside;
    return v > 0 ? kZoneAbove : kZoneBelow;
}

/// classify_transition with phase Normal folded in by the caller.
__device__ __forceinline__ int classify(int prev, int next, int direction) {
    if (prev == kZoneAbove) {
        if (next == kZoneBelow && direction <= 0) return kKindAcross;
        if (next == kZoneInside && direction <= 0) return kKindEntered;
        return kKindNone;
    }
    if (prev == kZoneBelow) {
        if (next == kZoneAbove && direction >= 0) return kKindAcross;
        if (next == kZoneInside && direction >= 0) return kKindEntered;
        return kKindNone;
    }
    return kKindNone;
}

/// Hands out the next system index; lanes arriving together share one
/// atomic (warp-aggregated through the coalesced group).
__device__ __forceinline__ Index fetch_system(unsigned long long* work) {
    namespace cg = cooperative_groups;
    cg::coalesced_group g = cg::coalesced_threads();
    unsigned long long base = 0;
    if (g.thread_rank() == 0) base = atomicAdd(work, static_cast<unsigned long long>(g.size()));
    base = g.shfl(base, 0);
    return static_cast<Index>(base + g.thread_rank());
}

enum Phase : int { kFetch = 0, kStep = 1, kSecant = 2, kCommit = 3, kFinish = 4, kDone = 5 };

constexpr int kMaxSecantIterations = 50; // events.hpp:190

/// The ensemble kernel. One instantiation per (model, algorithm): hooks are
/// inlined, widths are compile-time, all per-system state is in registers.
template <class H, Algorithm ALG>
__device__ __forceinline__ void solve_lanes(const H& m, const BatchArrays& b, const Controls& c) {
    constexpr int N = H::kSystemDim;
    constexpr int P = H::kParamCount > 0 ? H::kParamCount : 1;
    constexpr int E = H::kEventCount;
    constexpr int EE = E > 0 ? E : 1;
    constexpr int A = H::kAccessoryCount > 0 ? H::kAccessoryCount : 1;
    constexpr int NP = H::kParamCount, NA = H::kAccessoryCount;
    static_assert(N <= kMaxDim && E <= kMaxEvents, "model wider than the device controls");
    const Index n = b.n;

    // ---- per-lane registers
    Index sys = -1;
    Real td[2], y[N], p[P], acc[A];
    Real t = 0, t1 = 0, h = 0;
    // event machine (events.hpp:76-178)
    Real prev_value[EE];
    Index counter[EE];
    bool leaving[EE];
    Index steps_in_zone = 0;
    // outcome (driver.hpp:34-42)
    Index n_acc = 0, n_rej = 0, n_det = 0, n_secf = 0;
    Real smallest = 0;
    std::uint8_t reason = 0;
    // the step in flight
    Real h_try = 0, h_next = 0, h_step = 0, t_land = 0;
    bool clipped = false, relocated = false;
    int located = -1;
    Real y_land[N], f_land[EE];
    // secant (events.hpp:200-241)
    int s_idx = 0, s_it = 0;
    bool s_conv = false;
    Real th_prev = 0, f_prev = 0, th_cur = 0, f_cur = 0, th_min = 0, b_th = 0, b_f = 0;

    int phase = kFetch;

    const auto S = [](Real* a, int len) { return std::span<Real>(a, static_cast<std::size_t>(len)); };
    const auto CS = [](const Real* a, int len) { return std::span<const Real>(a, static_cast<std::size_t>(len)); };

    // Ends a secant location (driver.hpp:157-164).
    const auto end_secant = [&]() {
        if (!s_conv) ++n_secf;
        relocated = b_th < h_try;
        t_land = (clipped && !relocated) ? t1 : t + b_th;
        m.event_values(t_land, CS(y_land, N), CS(p, NP), S(f_land, E));
        phase = kCommit;
    };

    for (;;) {
        // ================= PREPARE: bring this lane to a pending RK evaluation
        for (;;) {
            if (phase == kFetch) {
                sys = fetch_system(b.work);
                if (sys >= n) {
                    phase = kDone;
                    break;
                }
                if (b.reason[sys] == static_cast<std::uint8_t>(StopReason::NonFiniteAbort)) continue; // solve.hpp:98
                td[0] = b.td[sys];
                td[1] = b.td[sys + n];
#pragma unroll
                for (int i = 0; i < N; ++i) y[i] = b.state[sys + i * n];
#pragma unroll
                for (int i = 0; i < H::kParamCount; ++i) p[i] = __ldg(b.params + sys + i * n);
#pragma unroll
                for (int i = 0; i < H::kAccessoryCount; ++i) acc[i] = b.acc[sys + i * n];
                n_acc = n_rej = n_det = n_secf = 0;
                smallest = __longlong_as_double(0x7ff0000000000000LL); // +inf
                reason = static_cast<std::uint8_t>(StopReason::ReachedEndTime);
                // driver.hpp:96-107
                m.initialize(td[0], S(td, 2), S(y, N), CS(p, NP), S(acc, NA));
                t = td[0];
                t1 = td[1];
                if constexpr (E > 0) {
                    Real f0[EE];
                    m.event_values(t, CS(y, N), CS(p, NP), S(f0, E));
#pragma unroll
                    for (int i = 0; i < E; ++i) {
                        prev_value[i] = f0[i];
                        leaving[i] = zone_of(f0[i], c.tolerance[i]) == kZoneInside;
                        counter[i] = 0;
                    }
                    steps_in_zone = 0;
                }
                h = ALG == Algorithm::RK4 ? c.initial_time_step
                                         : sclamp(c.initial_time_step, c.min_step, c.max_step);
                phase = kStep;
            }
            if (phase == kCommit) {
                // driver.hpp:170-227
                if (t_land <= t) {
                    reason = static_cast<std::uint8_t>(StopReason::NonFiniteAbort);
                    phase = kFinish;
                } else {
                    const Real advanced = t_land - t;
#pragma unroll
                    for (int i = 0; i < N; ++i) y[i] = y_land[i];
                    t = t_land;
                    ++n_acc;
                    smallest = smin(smallest, advanced);
                    bool event_stop = false;
                    if constexpr (E > 0) {
                        bool det[EE];
#pragma unroll
                        for (int i = 0; i < E; ++i) { // EventMachine::commit, events.hpp:134-156
                            const int pz = zone_of(prev_value[i], c.tolerance[i]);
                            const int nz = zone_of(f_land[i], c.tolerance[i]);
                            const bool kind = pz != kZoneNone && nz != kZoneNone && !leaving[i] &&
                                              classify(pz, nz, c.direction[i]) != kKindNone;
                            det[i] = kind || i == located;
                            if (det[i]) {
                                ++counter[i];
                                ++n_det;
                            }
                        }
                        Real f_post[EE];
                        if (located >= 0) {
#pragma unroll
                            for (int i = 0; i < E; ++i)
                                if (i == located) m.event_action(i, counter[i], t, S(y, N), CS(p, NP));
                            m.event_values(t, CS(y, N), CS(p, NP), S(f_post, E));
                        } else {
#pragma unroll
                            for (int i = 0; i < E; ++i) f_post[i] = f_land[i];
                        }
                        bool any_inside = false; // EventMachine::refresh, events.hpp:160-173
#pragma unroll
                        for (int i = 0; i < E; ++i) {
                            const int z = zone_of(f_post[i], c.tolerance[i]);
                            if (z == kZoneNone) continue;
                            prev_value[i] = f_post[i];
                            leaving[i] = z == kZoneInside;
                            any_inside = any_inside || z == kZoneInside;
                        }
                        steps_in_zone = any_inside ? steps_in_zone + 1 : 0;
#pragma unroll
                        for (int i = 0; i < E; ++i)
                            if (det[i]) m.event_accessory(i, counter[i], t, CS(y, N), CS(p, NP), S(acc, NA));
#pragma unroll
                        for (int i = 0; i < E; ++i)
                            if (det[i] && c.stop_condition[i] != 0 && counter[i] >= c.stop_condition[i])
                                event_stop = true;
                    }
                    m.ordinary_accessory(t, CS(y, N), CS(p, NP), S(acc, NA));
                    if (event_stop) {
                        reason = static_cast<std::uint8_t>(StopReason::EventStop);
                        phase = kFinish;
                    } else if (E > 0 && steps_in_zone >= c.max_steps_in_zone) {
                        reason = static_cast<std::uint8_t>(StopReason::EquilibriumStop);
                        phase = kFinish;
                    } else {
                        if (ALG == Algorithm::RKCK45 && !relocated) h = h_next;
                        phase = kStep;
                    }
                }
            }
            if (phase == kFinish) {
                // driver.hpp:231-233, then scatter_system (batch.cpp:32-40)
                m.finalize(t, S(td, 2), S(y, N), CS(p, NP), S(acc, NA));
                b.td[sys] = td[0];
                b.td[sys + n] = td[1];
#pragma unroll
                for (int i = 0; i < N; ++i) b.state[sys + i * n] = y[i];
#pragma unroll
                for (int i = 0; i < H::kAccessoryCount; ++i) b.acc[sys + i * n] = acc[i];
                b.final_t[sys] = t;
                b.reason[sys] = reason;
                b.accepted[sys] = n_acc;
                b.rejected[sys] = n_rej;
                b.detections[sys] = n_det;
                b.secant_failures[sys] = n_secf;
                b.smallest_step[sys] = smallest;
                phase = kFetch;
                continue;
            }
            if (phase == kStep) {
                // driver.hpp:109-119
                if (!(t < t1)) {
                    phase = kFinish;
                    continue;
                }
                h_try = h;
                clipped = false;
                if (t + h_try >= t1) {
                    h_try = t1 - t;
                    clipped = true;
                }
                if (!(h_try > 0)) {
                    t = t1;
                    phase = kFinish;
                    continue;
                }
                h_step = h_try;
                break;
            }
            if (phase == kSecant) {
                // events.hpp:214-219: the pre-step exits of one secant iteration
                if (s_it > kMaxSecantIterations) {
                    end_secant();
                    continue;
                }
                const Real denom = f_cur - f_prev;
                if (denom == 0) {
                    end_secant();
                    continue;
                }
                Real theta = th_cur - f_cur * (th_cur - th_prev) / denom;
                if (!isfinite(theta)) {
                    end_secant();
                    continue;
                }
                theta = sclamp(theta, th_min, h_try);
                if (theta == th_cur) {
                    end_secant();
                    continue;
                }
                h_step = theta;
                break;
            }
        }
        if (phase == kDone) break;

        // ================= the shared Runge-Kutta evaluation
        Real yn[N], err[N];
        const bool nonfinite = rk_step<H, ALG>(m, t, h_step, y, p, yn, err);

        // ================= ABSORB
        if (phase == kStep) {
            if constexpr (ALG == Algorithm::RK4) {
                if (nonfinite) { // driver.hpp:124-128
                    reason = static_cast<std::uint8_t>(StopReason::NonFiniteAbort);
                    phase = kFinish;
                    continue;
                }
                h_next = h;
            } else {
                // error_ratio (steppers.hpp:154-163) + control_step (176-198)
                Real ratio = 0.0;
#pragma unroll
                for (int i = 0; i < N; ++i) {
                    const Real scale = c.abs_tol[i] + c.rel_tol[i] * smax(fabs(y[i]), fabs(yn[i]));
                    ratio = smax(ratio, err[i] / scale);
                }
                bool accepted;
                if (nonfinite) {
                    if (h_try <= c.min_step) {
                        reason = static_cast<std::uint8_t>(StopReason::NonFiniteAbort);
                        phase = kFinish;
                        continue;
                    }
                    accepted = false;
                    h_next = smax(h_try * c.step_shrink_limit, c.min_step);
                } else {
                    accepted = ratio <= 1.0;
                    Real factor = 0.9 * pow(ratio, -0.2);
                    factor = sclamp(factor, c.step_shrink_limit, c.step_grow_limit);
                    h_next = sclamp(h_try * factor, c.min_step, c.max_step);
                    if (!accepted && h_try <= c.min_step) {
                        accepted = true;
                        h_next = c.min_step;
                    }
                }
                if (!accepted) {
                    ++n_rej;
                    h = h_next;
                    continue;
                }
            }
            // accepted: driver.hpp:146-168
            t_land = clipped ? t1 : t + h_try;
#pragma unroll
            for (int i = 0; i < N; ++i) y_land[i] = yn[i];
            located = -1;
            relocated = false;
            phase = kCommit;
            if constexpr (E > 0) {
                m.event_values(t_land, CS(y_land, N), CS(p, NP), S(f_land, E));
                // EventMachine::peek (events.hpp:111-125): highest index wins
                bool needs = false;
#pragma unroll
                for (int i = E - 1; i >= 0; --i) {
                    if (located >= 0) break;
                    const int pz = zone_of(prev_value[i], c.tolerance[i]);
                    const int nz = zone_of(f_land[i], c.tolerance[i]);
                    if (pz == kZoneNone || nz == kZoneNone || leaving[i]) continue;
                    const int kind = classify(pz, nz, c.direction[i]);
                    if (kind != kKindNone) {
                        located = i;
                        needs = kind == kKindAcross;
                    }
                }
                if (located >= 0 && needs) {
                    // start locate_secant (events.hpp:207-212); y_land holds y(h)
                    s_idx = located;
                    s_it = 1;
                    s_conv = false;
                    th_prev = 0;
                    th_cur = h_try;
                    th_min = h_try * 1e-12;
#pragma unroll
                    for (int i = 0; i < E; ++i)
                        if (i == s_idx) {
                            f_prev = prev_value[i];
                            f_cur = f_land[i];
                        }
                    b_th = h_try;
                    b_f = f_cur;
                    phase = kSecant;
                }
            }
        } else { // kSecant: one secant iteration's step is in (events.hpp:222-240)
            if constexpr (E > 0) {
                Real fs[EE];
                m.event_values(t + h_step, CS(yn, N), CS(p, NP), S(fs, E));
                Real f = fs[0];
                Real tol = c.tolerance[0];
#pragma unroll
                for (int i = 1; i < E; ++i)
                    if (i == s_idx) {
                        f = fs[i];
                        tol = c.tolerance[i];
                    }
                if (!isfinite(f)) {
                    end_secant();
                    continue;
                }
                if (fabs(f) < fabs(b_f)) {
                    b_th = h_step;
                    b_f = f;
#pragma unroll
                    for (int i = 0; i < N; ++i) y_land[i] = yn[i];
                }
                if (fabs(f) <= tol) {
                    s_conv = true;
                    end_secant();
                    continue;
                }
                th_prev = th_cur;
                f_prev = f_cur;
                th_cur = h_step;
                f_cur = f;
                ++s_it;
            }
        }
    }
}

template <class H, Algorithm ALG, int BLOCK, int MIN_BLOCKS>
__global__ void __launch_bounds__(BLOCK, MIN_BLOCKS) solve_kernel(H model, BatchArrays b, Controls c) {
    solve_lanes<H, ALG>(model, b, c);
}

} // namespace odegpu::device

#endif
