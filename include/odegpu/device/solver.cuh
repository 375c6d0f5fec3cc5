// solver.cuh — the sm_100a ensemble kernel: one thread integrates one system
// at a time, its hot state in registers; a lane that finishes its system fetches
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

#include <concepts>
#include <cstddef>
#include <cstdint>
#include <span>
#include <type_traits>

#include "odegpu.h"
#include "odegpu/device/dmath.cuh"
#include "odegpu/hooks.hpp"
#include "odegpu/trig.hpp"

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
    // classify_transition per event as a table: 2 bits (kind + 1) for each
    // (previous zone, next zone) pair, built from `direction` on the host
    // (controls_from), so the per-step peek is a shift and a mask
    unsigned kind_lut[kMaxEvents];
    Index max_steps_in_zone;
};

/// The streaming gate (odegpu_pipeline STREAMING, csrc/pipeline.cu): the
/// pool arrives in granules of 2^shift systems while the kernel runs. A lane
/// takes up system s only once *ready > s >> shift (the copy-in stream
/// bumps it after each granule group's H2D) and counts s when it is
/// finished, into done[group_of[granule]] — one counter (and one stream
/// wait) per copy-out group — which releases that group's D2H on the
/// copy-out stream. bad: [0] lowest index with t1 < t0 (~0: none), [2]
/// nonzero: aborted by the host or timed out. packed: every finished
/// system's outcome record in the reference's 56-byte AoS layout
/// (odegpu_outcome = SystemOutcome, driver.hpp:34-42), so the D2H ships
/// records without a packing pass.
struct StreamGate {
    const unsigned* ready = nullptr;
    unsigned* done = nullptr;             // per copy-out group (group_of[granule])
    const unsigned short* group_of = nullptr;
    unsigned long long* bad = nullptr;
    unsigned char* packed = nullptr;
    unsigned shift = 0;
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
    Index n;                  // stride (batch capacity)
    Index count;              // systems [0, count) are integrated (count <= n)
    unsigned long long* work; // next system to hand out (zeroed before launch)
    // fetch order: the j-th system handed out is order[j] (a permutation of
    // [0, count)), or j when null (odegpu_batch_set_fetch_order)
    const unsigned* order = nullptr;
    // when non-null: each finished system's RK evaluations (trial steps +
    // secant re-steps), the key of the next fetch order
    unsigned* cost = nullptr;
    // Fused iterations: every system is solved `iterations` times in a row
    // by the lane that took it up (solve_iteratively without a sink, models
    // with kFusableIterations); 1 = one solve per launch.
    int iterations = 1;
    // When non-null: trial steps (accepted + rejected) of every system and
    // iteration the launch integrates are added here (one atomic per warp).
    unsigned long long* trial_steps = nullptr;
    // Scan tallies (ScanDiagnostics, scan.hpp:41-49), accumulated across
    // solves when non-null: [5] detections, [6] detections outside their
    // zone, [7] max |F|/tolerance over detections (bits of a non-negative
    // double), [8] systems whose t0 did not advance over the solve (kTally*).
    unsigned long long* tally = nullptr;
    // Per-detection log (the reference's on_detection observer,
    // solve.hpp:46-50 / driver.hpp:186-206), when non-null: one record per
    // committed detection, appended at slot atomicAdd(log_count, 1) while
    // slots last (later ones are only counted). SoA columns of log_capacity.
    unsigned long long* log_count = nullptr;
    Index log_capacity = 0;
    unsigned* log_system = nullptr;          // batch index
    int* log_event = nullptr;                // event index
    int* log_kind = nullptr;                 // DetectionKind (events.hpp:31)
    int* log_in_zone = nullptr;
    long long* log_counter = nullptr;        // Detection::counter (1-based)
    long long* log_sequence = nullptr;       // the system's detection number in this solve
    Real* log_t = nullptr;
    Real* log_value = nullptr;
    Real* log_y_pre = nullptr;               // [dim][capacity]: state before event_action
    Real* log_y_post = nullptr;              // [dim][capacity]: state after it
    // When non-null: every finished system's outcome record in the
    // reference's 56-byte AoS layout (odegpu_outcome = SystemOutcome,
    // driver.hpp:34-42), written next to the SoA fields at finish, so a
    // pipeline ships records to the host without a packing pass.
    unsigned char* packed = nullptr;
    // Streaming pool (odegpu_pipeline, streaming mode, csrc/pipeline.cu;
    // the STREAM instantiation only): the pool's granules land while the
    // kernel runs — StreamGate.
    StreamGate gate{};
};

/// kStreamAbort in *gate.ready: the host abandoned the run. A lane that
/// waits longer than kStreamTimeoutNs for a granule gives up (bad[2]);
/// either way every system is still counted done, so no copy-out wait is
/// left hanging.
constexpr unsigned kStreamAbort = 0x80000000u;
constexpr unsigned long long kStreamTimeoutNs = 20ull * 1000 * 1000 * 1000;

__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ unsigned ld_relaxed_gpu(const unsigned* p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

/// Counts a finished (or skipped) system into its granule with release
/// semantics (MEMBAR.ALL.GPU + REDG; __threadfence would be MEMBAR.SC plus
/// an L1 invalidation): the system's stores are visible before the count
/// the copy-out stream waits on.
__device__ __forceinline__ void stream_release(const StreamGate& g, unsigned sys) {
    unsigned* const d = g.done + __ldg(g.group_of + (sys >> g.shift));
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(d) : "memory");
}

/// Per-block shared state of the STREAM instantiation: [0, BLOCK) each
/// lane's finished system whose count is still pending (+1; 0 = none),
/// [BLOCK] the highest granule count any lane of the block has seen land.
template <bool STREAM, int BLOCK>
__device__ __forceinline__ unsigned* stream_shared() {
    if constexpr (STREAM) {
        __shared__ unsigned s[BLOCK + 1];
        return s;
    } else {
        return nullptr;
    }
}

/// Waits until the granule holding system `sys` has landed; false when the
/// run was aborted or the wait timed out (the caller counts the system done
/// and skips it).
///
/// The common case costs no global load: the block remembers the highest
/// granule count it has seen (`landed`, shared memory). Otherwise one
/// relaxed load — an acquire would invalidate the SM's whole L1 (CCTL.IVALL
/// in the SASS). That is safe because no L1 can hold a stale line of a
/// granule: granules are 2^k >= 32 systems, so every 128-byte line of every
/// SoA array lies in one granule, and no lane loads a line of a granule
/// before it has seen that granule land (the loads are control-dependent on
/// the flag). A lane that had to wait takes one acquire load at the end.
__device__ __forceinline__ bool stream_wait(const StreamGate& g, unsigned* landed, unsigned sys) {
    const unsigned need = (sys >> g.shift) + 1u;
    if (need <= *reinterpret_cast<volatile unsigned*>(landed)) return true;
    unsigned v = ld_relaxed_gpu(g.ready);
    unsigned long long t0 = 0;
    bool waited = false;
    for (;;) {
        if (v & kStreamAbort) return false;
        if (v >= need) break;
        waited = true;
        if (*reinterpret_cast<volatile unsigned long long*>(g.bad + 2)) return false;
        const unsigned long long now = global_ns();
        if (t0 == 0) {
            t0 = now;
        } else if (now - t0 > kStreamTimeoutNs) {
            atomicOr(g.bad + 2, 1ull);
            return false;
        }
        __nanosleep(400);
        v = ld_relaxed_gpu(g.ready);
    }
    if (waited) v = ld_acquire_gpu(g.ready) & ~kStreamAbort;
    atomicMax(landed, v);
    return true;
}

/// A streaming run's end of one system: its AoS outcome record (when the
/// run ships outcomes). Its count into the granule follows at the lane's
/// next fetch (the release fence then finds these stores long performed
/// instead of stalling the warp on them).
static __device__ __forceinline__ void stream_finish(const StreamGate& g, unsigned sys, Real final_t, unsigned reason,
                                                     Index acc, Index rej, Index det, Index secf, Real smallest) {
    if (g.packed) {
        unsigned long long* r = reinterpret_cast<unsigned long long*>(g.packed + static_cast<std::size_t>(sys) * 56);
        r[0] = static_cast<unsigned long long>(__double_as_longlong(final_t));
        r[1] = reason; // the reason byte and 7 zero pad bytes (little-endian)
        r[2] = static_cast<unsigned long long>(acc);
        r[3] = static_cast<unsigned long long>(rej);
        r[4] = static_cast<unsigned long long>(det);
        r[5] = static_cast<unsigned long long>(secf);
        r[6] = static_cast<unsigned long long>(__double_as_longlong(smallest));
    }
}

/// Slots of the scan tally (shared with the tally kernel, csrc/kernels.cu).
enum : int {
    kTallyReason0 = 0, kTallySecantFailures = 4, kTallyDetections = 5, kTallyOutsideZone = 6,
    kTallyMaxRatio = 7, kTallyStartNotAdvanced = 8, kTallyNonfinite = 9, kTallySlots = 10
};

// --- Cash-Karp tableau (steppers.hpp:16-39): exact rationals rendered once.
namespace ckv {
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
} // namespace ckv

/// The same values as the kernels read them: coefficients with long
/// mantissas live in the constant bank, so ptxas folds them into c[][]
/// operands of the DFMAs instead of two UMOVs per use; short ones (1, 7/8,
/// 5/2) stay encodable immediates.
namespace ck {
static __constant__ Real c2 = ckv::c2, c3 = ckv::c3, c4 = ckv::c4;
constexpr Real c5 = ckv::c5, c6 = ckv::c6;
static __constant__ Real a21 = ckv::a21, a31 = ckv::a31, a32 = ckv::a32, a41 = ckv::a41, a42 = ckv::a42,
                         a43 = ckv::a43, a51 = ckv::a51, a53 = ckv::a53, a54 = ckv::a54, a61 = ckv::a61,
                         a62 = ckv::a62, a63 = ckv::a63, a64 = ckv::a64, a65 = ckv::a65;
constexpr Real a52 = ckv::a52;
static __constant__ Real b1 = ckv::b1, b3 = ckv::b3, b4 = ckv::b4, b6 = ckv::b6;
static __constant__ Real d1 = ckv::d1, d3 = ckv::d3, d4 = ckv::d4, d5 = ckv::d5, d6 = ckv::d6;
} // namespace ck

// std::max / std::min / std::clamp semantics, including NaN behaviour.
__device__ __forceinline__ Real smax(Real a, Real b) { return (a < b) ? b : a; }
__device__ __forceinline__ Real smin(Real a, Real b) { return (b < a) ? b : a; }
__device__ __forceinline__ Real sclamp(Real v, Real lo, Real hi) { return (v < lo) ? lo : (hi < v) ? hi : v; }

/// Compiler-level memory fence: nothing cached from shared memory survives
/// it in registers (keeps cold state and shared-memory parameters out of the
/// register file across the RK stages).
__device__ __forceinline__ void cold_fence() { asm volatile("" ::: "memory"); }

/// A state vector passed by value (registers) through an outlined RHS call.
template <int N>
struct StateVec {
    Real v[N];
};

/// The model's RHS as a real (non-inlined) device function: its register
/// allocation is its own, not interleaved with the step loop's. For a large
/// RHS (Keller-Miksis) this is what lets straight-line stages stay small in
/// code and in registers.
template <class H>
__device__ __noinline__ StateVec<H::kSystemDim> rhs_outline(const H m, Real t, StateVec<H::kSystemDim> y,
                                                            const Real* p) {
    StateVec<H::kSystemDim> dy;
    m.ode_rhs(t, std::span<const Real>(y.v, H::kSystemDim), std::span<const Real>(p, H::kParamCount),
              std::span<Real>(dy.v, H::kSystemDim));
    return dy;
}

template <class H, bool OUTLINE = false>
__device__ __forceinline__ void rhs(const H& m, Real t, const Real (&y)[H::kSystemDim],
                                    const Real* p, Real (&dy)[H::kSystemDim]) {
    if constexpr (OUTLINE) {
        StateVec<H::kSystemDim> in;
#pragma unroll
        for (int i = 0; i < H::kSystemDim; ++i) in.v[i] = y[i];
        const StateVec<H::kSystemDim> out = rhs_outline<H>(m, t, in, p);
#pragma unroll
        for (int i = 0; i < H::kSystemDim; ++i) dy[i] = out.v[i];
    } else {
        m.ode_rhs(t, std::span<const Real>(y, H::kSystemDim), std::span<const Real>(p, H::kParamCount),
                  std::span<Real>(dy, H::kSystemDim));
    }
}

/// Number of cached time terms of a model (hooks.hpp TimeSplitHooks), 0 if
/// it does not split its RHS.
template <class H>
inline constexpr int kTimeTerms = [] {
    if constexpr (TimeSplitHooks<H>) return static_cast<int>(H::kTimeTermCount);
    else return 0;
}();

/// The outlined halves of a time-split model's RHS: its time terms, and the
/// RHS given them.
template <class H>
__device__ __noinline__ StateVec<kTimeTerms<H>> time_terms_outline(const H m, Real t, const Real* p) {
    StateVec<kTimeTerms<H>> tt;
    m.time_terms(t, std::span<const Real>(p, H::kParamCount), std::span<Real>(tt.v, kTimeTerms<H>));
    return tt;
}
template <class H>
__device__ __noinline__ StateVec<H::kSystemDim> rhs_split_outline(const H m, Real t, StateVec<H::kSystemDim> y,
                                                                  const Real* p, StateVec<kTimeTerms<H>> tt) {
    StateVec<H::kSystemDim> dy;
    m.ode_rhs_split(t, std::span<const Real>(y.v, H::kSystemDim), std::span<const Real>(p, H::kParamCount),
                    std::span<const Real>(tt.v, kTimeTerms<H>), std::span<Real>(dy.v, H::kSystemDim));
    return dy;
}

/// One RHS evaluation of a time-split model at stage time t: the time terms
/// tt are computed when `need` (and returned in tt), reused otherwise.
template <class H, bool OUTLINE>
__device__ __forceinline__ void rhs_tt(const H& m, Real t, const Real (&y)[H::kSystemDim], const Real* p,
                                       Real (&tt)[kTimeTerms<H>], bool need, Real (&dy)[H::kSystemDim]) {
    constexpr int N = H::kSystemDim, K = kTimeTerms<H>;
    if constexpr (OUTLINE) {
        StateVec<K> tin;
        if (need) {
            tin = time_terms_outline<H>(m, t, p);
        } else {
#pragma unroll
            for (int i = 0; i < K; ++i) tin.v[i] = tt[i];
        }
        StateVec<N> in;
#pragma unroll
        for (int i = 0; i < N; ++i) in.v[i] = y[i];
        const StateVec<N> out = rhs_split_outline<H>(m, t, in, p, tin);
#pragma unroll
        for (int i = 0; i < N; ++i) dy[i] = out.v[i];
#pragma unroll
        for (int i = 0; i < K; ++i) tt[i] = tin.v[i];
    } else {
        if (need) m.time_terms(t, std::span<const Real>(p, H::kParamCount), std::span<Real>(tt, K));
        m.ode_rhs_split(t, std::span<const Real>(y, N), std::span<const Real>(p, H::kParamCount),
                        std::span<const Real>(tt, K), std::span<Real>(dy, N));
    }
}

/// A stage evaluation that does not touch the time-term cache.
template <class H, bool OUTLINE>
__device__ __forceinline__ void rhs_stage(const H& m, Real t, const Real (&y)[H::kSystemDim], const Real* p,
                                          Real (&dy)[H::kSystemDim]) {
    rhs<H, OUTLINE>(m, t, y, p, dy);
}

/// One trial step from (t, y) with step h (steppers.hpp:82-139). Writes the
/// proposed state, the embedded error |y5 - y4| (RKCK45) and whether
/// anything is non-finite. Expressions are those of the reference, operation
/// for operation — but the default build lets nvcc contract a*b+c into one
/// DFMA (one rounding instead of two), which the reference's g++ build
/// without -march never does; only the parity build (make parity,
/// -fmad=false) rounds every product and sum separately like the reference.
///
/// ROLLED: the stages are a rolled loop around ONE inlined RHS call site; a
/// uniform switch on the stage index forms the stage argument from the
/// tableau row, so a large RHS (libdevice pow / sincos for Keller-Miksis) is
/// emitted once instead of 4-6 times and the step loop fits the instruction
/// cache. Every lane of a warp runs the same stage, so the switch never
/// diverges. The stage derivatives of the rolled loop live in shared memory
/// (kb: this thread's column, stride BLOCK — conflict-free): a loop-carried
/// k1..k5 in registers costs ~20 registers across the RHS plus register
/// moves at every stage, while the smem form costs ~40 LDS/STS per step.
///
/// Time-split models (kTimeTerms<H> > 0, straight-line stages) go through
/// the lane's time-term cache `tc` (TimeTermCache): the first stage reuses
/// the cached terms when their time equals t, and the step leaves the terms
/// at its end point t + h behind (the next step's start once accepted; a
/// two-slot policy also keeps those at t for a rejected step's retry).
template <class H, Algorithm ALG, bool ROLLED, int BLOCK, bool OUTLINE, class TC>
__device__ __forceinline__ bool rk_step(const H& m, Real t, Real h, const Real (&y)[H::kSystemDim],
                                        const Real* p, Real (&out)[H::kSystemDim],
                                        Real (&err)[H::kSystemDim], Real* kb, const TC& tc) {
    constexpr int N = H::kSystemDim;
    constexpr int K = kTimeTerms<H>;
    bool finite = true;
    // the first stage and the stage at t + h through the time-term cache
    const auto first = [&](Real (&dy)[N]) {
        if constexpr (TC::kEnabled && K > 0 && !ROLLED) {
            Real tt[K];
            const bool hit = tc.lookup(t, tt);
            rhs_tt<H, OUTLINE>(m, t, y, p, tt, !hit, dy);
            tc.store(0, t, tt);
        } else {
            rhs_stage<H, OUTLINE>(m, t, y, p, dy);
        }
    };
    const auto at_end = [&](const Real (&ys)[N], Real (&dy)[N]) {
        if constexpr (TC::kEnabled && K > 0 && !ROLLED) {
            Real tt[K];
            rhs_tt<H, OUTLINE>(m, t + h, ys, p, tt, true, dy);
            tc.store(1, t + h, tt);
        } else {
            rhs_stage<H, OUTLINE>(m, t + h, ys, p, dy);
        }
    };
    if constexpr (!ROLLED) {
        // Straight-line stages: best when the RHS is small (Duffing, valve):
        // no stage dispatch, the scheduler sees across stage boundaries.
        Real k1[N], k2[N], k3[N], k4[N], k5[N], k6[N];
        Real yt[N];
        if constexpr (ALG == Algorithm::RK4) {
            first(k1);
#pragma unroll
            for (int i = 0; i < N; ++i) yt[i] = y[i] + 0.5 * h * k1[i];
            rhs_stage<H, OUTLINE>(m, t + 0.5 * h, yt, p, k2);
#pragma unroll
            for (int i = 0; i < N; ++i) yt[i] = y[i] + 0.5 * h * k2[i];
            rhs_stage<H, OUTLINE>(m, t + 0.5 * h, yt, p, k3);
#pragma unroll
            for (int i = 0; i < N; ++i) yt[i] = y[i] + h * k3[i];
            at_end(yt, k4);
#pragma unroll
            for (int i = 0; i < N; ++i) {
                out[i] = y[i] + (h / 6.0) * (k1[i] + 2.0 * k2[i] + 2.0 * k3[i] + k4[i]);
                err[i] = 0.0;
                finite = finite && isfinite(out[i]);
            }
        } else {
            first(k1);
#pragma unroll
            for (int i = 0; i < N; ++i) yt[i] = y[i] + h * (ck::a21 * k1[i]);
            rhs_stage<H, OUTLINE>(m, t + ck::c2 * h, yt, p, k2);
#pragma unroll
            for (int i = 0; i < N; ++i) yt[i] = y[i] + h * (ck::a31 * k1[i] + ck::a32 * k2[i]);
            rhs_stage<H, OUTLINE>(m, t + ck::c3 * h, yt, p, k3);
#pragma unroll
            for (int i = 0; i < N; ++i) yt[i] = y[i] + h * (ck::a41 * k1[i] + ck::a42 * k2[i] + ck::a43 * k3[i]);
            rhs_stage<H, OUTLINE>(m, t + ck::c4 * h, yt, p, k4);
#pragma unroll
            for (int i = 0; i < N; ++i)
                yt[i] = y[i] + h * (ck::a51 * k1[i] + ck::a52 * k2[i] + ck::a53 * k3[i] + ck::a54 * k4[i]);
            static_assert(ck::c5 == 1.0, "Cash-Karp stage 5 is the step's end point");
            at_end(yt, k5);
#pragma unroll
            for (int i = 0; i < N; ++i)
                yt[i] = y[i] + h * (ck::a61 * k1[i] + ck::a62 * k2[i] + ck::a63 * k3[i] + ck::a64 * k4[i] +
                                    ck::a65 * k5[i]);
            rhs_stage<H, OUTLINE>(m, t + ck::c6 * h, yt, p, k6);
#pragma unroll
            for (int i = 0; i < N; ++i) {
                out[i] = y[i] + h * (ck::b1 * k1[i] + ck::b3 * k3[i] + ck::b4 * k4[i] + ck::b6 * k6[i]);
                err[i] = fabs(h * (ck::d1 * k1[i] + ck::d3 * k3[i] + ck::d4 * k4[i] + ck::d5 * k5[i] +
                                   ck::d6 * k6[i]));
                finite = finite && isfinite(out[i]) && isfinite(err[i]);
            }
        }
        return !finite;
    }
    // rolled: k_s (s = 1..STAGES-1) in shared memory, the last one in registers
#define ODEGPU_K(s, i) kb[((s) - 1) * N * BLOCK + (i) * BLOCK]
    Real kk[N];
    if constexpr (ALG == Algorithm::RK4) {
#pragma unroll 1
        for (int s = 1; s <= 4; ++s) {
            cold_fence();
            Real ts, yt[N];
            switch (s) {
            case 1:
                ts = t;
#pragma unroll
                for (int i = 0; i < N; ++i) yt[i] = y[i];
                break;
            case 2:
                ts = t + 0.5 * h;
#pragma unroll
                for (int i = 0; i < N; ++i) yt[i] = y[i] + 0.5 * h * ODEGPU_K(1, i);
                break;
            case 3:
                ts = t + 0.5 * h;
#pragma unroll
                for (int i = 0; i < N; ++i) yt[i] = y[i] + 0.5 * h * ODEGPU_K(2, i);
                break;
            default:
                ts = t + h;
#pragma unroll
                for (int i = 0; i < N; ++i) yt[i] = y[i] + h * ODEGPU_K(3, i);
                break;
            }
            rhs<H, OUTLINE>(m, ts, yt, p, kk);
            if (s < 4) {
#pragma unroll
                for (int i = 0; i < N; ++i) ODEGPU_K(s, i) = kk[i];
            }
        }
        cold_fence();
#pragma unroll
        for (int i = 0; i < N; ++i) {
            out[i] = y[i] + (h / 6.0) * (ODEGPU_K(1, i) + 2.0 * ODEGPU_K(2, i) + 2.0 * ODEGPU_K(3, i) + kk[i]);
            err[i] = 0.0;
            finite = finite && isfinite(out[i]);
        }
    } else {
#pragma unroll 1
        for (int s = 1; s <= 6; ++s) {
            cold_fence();
            Real ts, yt[N];
            switch (s) {
            case 1:
                ts = t;
#pragma unroll
                for (int i = 0; i < N; ++i) yt[i] = y[i];
                break;
            case 2:
                ts = t + ck::c2 * h;
#pragma unroll
                for (int i = 0; i < N; ++i) yt[i] = y[i] + h * (ck::a21 * ODEGPU_K(1, i));
                break;
            case 3:
                ts = t + ck::c3 * h;
#pragma unroll
                for (int i = 0; i < N; ++i) yt[i] = y[i] + h * (ck::a31 * ODEGPU_K(1, i) + ck::a32 * ODEGPU_K(2, i));
                break;
            case 4:
                ts = t + ck::c4 * h;
#pragma unroll
                for (int i = 0; i < N; ++i)
                    yt[i] = y[i] + h * (ck::a41 * ODEGPU_K(1, i) + ck::a42 * ODEGPU_K(2, i) + ck::a43 * ODEGPU_K(3, i));
                break;
            case 5:
                ts = t + ck::c5 * h;
#pragma unroll
                for (int i = 0; i < N; ++i)
                    yt[i] = y[i] + h * (ck::a51 * ODEGPU_K(1, i) + ck::a52 * ODEGPU_K(2, i) +
                                        ck::a53 * ODEGPU_K(3, i) + ck::a54 * ODEGPU_K(4, i));
                break;
            default:
                ts = t + ck::c6 * h;
#pragma unroll
                for (int i = 0; i < N; ++i)
                    yt[i] = y[i] + h * (ck::a61 * ODEGPU_K(1, i) + ck::a62 * ODEGPU_K(2, i) +
                                        ck::a63 * ODEGPU_K(3, i) + ck::a64 * ODEGPU_K(4, i) +
                                        ck::a65 * ODEGPU_K(5, i));
                break;
            }
            rhs<H, OUTLINE>(m, ts, yt, p, kk);
            if (s < 6) {
#pragma unroll
                for (int i = 0; i < N; ++i) ODEGPU_K(s, i) = kk[i];
            }
        }
        cold_fence();
#pragma unroll
        for (int i = 0; i < N; ++i) {
            out[i] = y[i] + h * (ck::b1 * ODEGPU_K(1, i) + ck::b3 * ODEGPU_K(3, i) + ck::b4 * ODEGPU_K(4, i) +
                                 ck::b6 * kk[i]);
            err[i] = fabs(h * (ck::d1 * ODEGPU_K(1, i) + ck::d3 * ODEGPU_K(3, i) + ck::d4 * ODEGPU_K(4, i) +
                               ck::d5 * ODEGPU_K(5, i) + ck::d6 * kk[i]));
            finite = finite && isfinite(out[i]) && isfinite(err[i]);
        }
    }
#undef ODEGPU_K
    return !finite;
}

// Event zones (events.hpp:22-26) and transitions (events.hpp:54-70). Zone
// codes fit two bits so a lane keeps zone_of(prev_value) of every event in
// one register. EventMachine's phase is implied: an event is Leaving exactly
// when its previous value sits inside the zone (init, events.hpp:93-101, and
// refresh, events.hpp:160-173, set both together), and classify_transition
// never fires from Inside, so the phase needs no storage of its own.
enum : int { kZoneBelow = 0, kZoneInside = 1, kZoneAbove = 2, kZoneNone = 3 };
enum : int { kKindNone = -1, kKindAcross = 0, kKindEntered = 1 };

/// events.hpp:22-33, as selects: it runs on every accepted step.
__device__ __forceinline__ int zone_of(Real v, Real tol) {
    const bool fin = fabs(v) < __longlong_as_double(0x7ff0000000000000LL); // false for inf and NaN
    int z = v > 0 ? kZoneAbove : kZoneBelow;
    z = fabs(v) <= tol ? kZoneInside : z;
    return fin ? z : kZoneNone;
}

/// classify_transition (events.hpp:54-70) from the previous zone; kZoneNone
/// on either side and Inside before (phase Leaving) give no detection.
/// (Host and device: controls_from tabulates it per event direction.)
__host__ __device__ constexpr int classify(int prev, int next, int direction) {
    if (prev == kZoneAbove && direction <= 0) {
        if (next == kZoneBelow) return kKindAcross;
        if (next == kZoneInside) return kKindEntered;
    }
    if (prev == kZoneBelow && direction >= 0) {
        if (next == kZoneAbove) return kKindAcross;
        if (next == kZoneInside) return kKindEntered;
    }
    return kKindNone;
}

/// classify() looked up in the event's table (Controls::kind_lut).
__device__ __forceinline__ int classify_lut(int prev, int next, unsigned lut) {
    return static_cast<int>((lut >> (2 * (4 * prev + next))) & 3u) - 1;
}
__host__ __device__ constexpr unsigned kind_table(int direction) {
    unsigned lut = 0;
    for (int prev = 0; prev < 4; ++prev)
        for (int next = 0; next < 4; ++next)
            lut |= static_cast<unsigned>(classify(prev, next, direction) + 1) << (2 * (4 * prev + next));
    return lut;
}

__device__ __forceinline__ int zone_at(int zones, int i) { return (zones >> (2 * i)) & 3; }
__device__ __forceinline__ int with_zone(int zones, int i, int z) {
    return (zones & ~(3 << (2 * i))) | (z << (2 * i));
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

/// Lane phases. Those below kReadyStep are bookkeeping run in the prepare
/// loop; kReadyStep / kReadySecant mean an RK evaluation of length h_step
/// from (t, y) is pending (a trial step, or one secant re-step).
enum Phase : int {
    kFetch = 0, kRefetch = 1, kSetup = 2, kSecant = 3, kCommit = 4, kFinish = 5, kDone = 6, kReadyStep = 7,
    kReadySecant = 8
};

constexpr int kMaxSecantIterations = 50; // events.hpp:190

/// Cold per-lane state: what only the infrequent paths touch (system
/// entry/exit, detections, the secant, accessories). It lives in shared
/// memory as structure of arrays (one column per thread, bank-conflict free)
/// so that only the hot set — t, h, y, the step bookkeeping and the stage
/// vectors — occupies registers; that is what sets occupancy.
template <class H, int BLOCK, int TT_SLOTS = 0>
struct ColdState {
    static constexpr int N = H::kSystemDim;
    static constexpr int E = H::kEventCount > 0 ? H::kEventCount : 1;
    static constexpr int A = H::kAccessoryCount > 0 ? H::kAccessoryCount : 1;
    Real td[2][BLOCK];
    Real acc[A][BLOCK];
    Real y_land[N][BLOCK];
    Real f_land[E][BLOCK];
    Real prev_value[E][BLOCK]; // EventMachine (events.hpp:76-178)
    Real h_try[BLOCK], h_next[BLOCK], t_land[BLOCK];
    unsigned long long lane_trial_steps[BLOCK]; // lane's trial steps (BatchArrays::trial_steps)
    Real lane_max_ratio[BLOCK];    // lane accumulators for the scan tally,
    unsigned lane_outside[BLOCK];  // over every system the lane integrates
    unsigned lane_not_advanced[BLOCK];
    unsigned lane_detections[BLOCK];
    // secant iterates (events.hpp:207-240); its lower bound h_try * 1e-12 is
    // recomputed from h_try (bitwise the same value) instead of stored
    Real th_prev[BLOCK], f_prev[BLOCK], th_cur[BLOCK], f_cur[BLOCK], b_th[BLOCK], b_f[BLOCK];
    unsigned sys[BLOCK]; // batch slot (batches hold < 2^32 systems, odegpu_batch_create)
    // SystemOutcome counters are int64 (driver.hpp:37-40): detections and
    // secant failures count in 64 bits here; the per-step accepted / rejected
    // counters (Bookkeeping) count in 32 bits and carry into these high words
    unsigned long long n_det[BLOCK], n_secf[BLOCK];
    unsigned acc_hi[BLOCK], rej_hi[BLOCK];
    // secant re-steps of the current system (its cost beyond the trial steps;
    // a fetch-order key, saturating) and the fused iterations still to run on
    // it (BatchArrays::iterations <= 65535 per launch): 16 bits each, so the
    // Keller-Miksis layout keeps its 5 blocks per SM
    unsigned short n_resteps[BLOCK], it_left[BLOCK];
    long long counter[E][BLOCK]; // EventMachine counters (events.hpp:87), Index in the reference
    // secant iteration (<= kMaxSecantIterations + 1), its event, the located
    // event (-1: none) and flags: bytes, so that the 64-bit counters above fit
    // the Keller-Miksis kernel's 5-blocks-per-SM shared-memory budget
    unsigned char s_it[BLOCK], s_idx[BLOCK];
    signed char located[BLOCK];
    unsigned char clipped[BLOCK], relocated[BLOCK], s_conv[BLOCK], reason[BLOCK];
    // time-term cache of a time-split model (rk_step): slot s holds the
    // terms at tt_key[s]
    static constexpr int TTB = TT_SLOTS > 0 ? BLOCK : 1;
    static constexpr int TTS = TT_SLOTS > 0 ? TT_SLOTS : 1;
    Real tt_key[TTS][TTB];
    Real tt_val[TTS][kTimeTerms<H> > 0 ? kTimeTerms<H> : 1][TTB];
};

/// A lane's view of its time-term cache (two slots in its ColdState column).
template <class CS, int K, bool ENABLED, int SLOTS = 1>
struct TimeTermCache {
    static constexpr bool kEnabled = ENABLED;
    CS& cs;
    int tid;
    // two slots: [0] the terms at the step's start t (first stage), [1] at
    // its end point t + h; one slot: only the end point, in [0]
    __device__ __forceinline__ bool lookup(Real t, Real (&tt)[K]) const {
        if constexpr (SLOTS == 1) {
#pragma unroll
            for (int i = 0; i < K; ++i) tt[i] = cs.tt_val[0][i][tid];
            return t == cs.tt_key[0][tid];
        } else {
            const bool in1 = t == cs.tt_key[1][tid];
#pragma unroll
            for (int i = 0; i < K; ++i) tt[i] = in1 ? cs.tt_val[1][i][tid] : cs.tt_val[0][i][tid];
            return in1 || t == cs.tt_key[0][tid];
        }
    }
    __device__ __forceinline__ void store(int slot, Real key, const Real (&tt)[K]) const {
        if constexpr (SLOTS == 1) {
            if (slot == 0) return;
            slot = 0;
        }
        cs.tt_key[slot][tid] = key;
#pragma unroll
        for (int i = 0; i < K; ++i) cs.tt_val[slot][i][tid] = tt[i];
    }
    __device__ __forceinline__ void clear() const {
#pragma unroll
        for (int s = 0; s < SLOTS; ++s) cs.tt_key[s][tid] = __longlong_as_double(0x7ff8000000000000LL); // NaN
    }
};

/// Per-step bookkeeping of a lane (t1, SystemOutcome counters, EventMachine
/// zones): read or written on every step, but not inside the RK stages.
template <int BLOCK>
struct Bookkeeping {
    Real t1[BLOCK];
    Real h[BLOCK];              // the driver's step size (driver.hpp:105)
    Real smallest[BLOCK];       // SystemOutcome::smallest_step
    unsigned n_acc[BLOCK], n_rej[BLOCK];
    int zones[BLOCK];           // zone_of(prev_value[i]), 2 bits per event
    int steps_in_zone[BLOCK];   // EventMachine::steps_in_zone_
};

/// Whether a model overrides a HookDefaults no-op (inherited hooks keep the
/// HookDefaults member-pointer type): per-step hooks that do nothing cost
/// nothing, not even the shared-memory traffic around them.
template <class H>
inline constexpr bool kHasOrdinaryAccessory = !std::is_same_v<decltype(&H::ordinary_accessory),
                                                              decltype(&HookDefaults::ordinary_accessory)>;

/// Per-model kernel structure, chosen from ncu measurements
/// and specialisable for custom models:
///  * kRolledStages   — one RHS call site in a rolled stage loop (pays off
///                      when the RHS is large: I-cache, registers);
///  * kColdInShared   — cold lane state in shared memory instead of registers;
///  * kParamsInShared — per-system parameters in shared memory (one row of
///                      odd stride per thread, conflict-free 8-byte loads);
///  * kBookInShared   — the per-step bookkeeping (Bookkeeping) in shared
///                      memory: a few LDS/STS per step for fewer registers
///                      across the stages (large RHS, high register demand);
///  * kOutlineRhs     — the RHS as a real call (rhs_outline) instead of
///                      inlined into each stage: a large RHS keeps its own
///                      register allocation and is emitted once.
/// ODEGPU_POLICY_{ROLLED,COLD_SHARED,PARAMS_SHARED} override every model in
/// tuning builds (scripts/build_variants.sh).
template <class H>
struct KernelPolicy {
    static constexpr bool kRolledStages = false;
    static constexpr bool kColdInShared = true;
    static constexpr bool kParamsInShared = false;
    static constexpr bool kBookInShared = false;
    static constexpr bool kOutlineRhs = false;
    static constexpr bool kCacheTimeTerms = true;
};

template <class H>
struct EffectivePolicy {
#ifdef ODEGPU_POLICY_ROLLED
    static constexpr bool kRolledStages = ODEGPU_POLICY_ROLLED;
#else
    static constexpr bool kRolledStages = KernelPolicy<H>::kRolledStages;
#endif
#ifdef ODEGPU_POLICY_COLD_SHARED
    static constexpr bool kColdInShared = ODEGPU_POLICY_COLD_SHARED;
#else
    static constexpr bool kColdInShared = KernelPolicy<H>::kColdInShared;
#endif
#ifdef ODEGPU_POLICY_PARAMS_SHARED
    static constexpr bool kParamsInShared = ODEGPU_POLICY_PARAMS_SHARED && H::kParamCount > 0;
#else
    static constexpr bool kParamsInShared = KernelPolicy<H>::kParamsInShared && H::kParamCount > 0;
#endif
#ifdef ODEGPU_POLICY_OUTLINE_RHS
    static constexpr bool kOutlineRhs = ODEGPU_POLICY_OUTLINE_RHS;
#else
    static constexpr bool kOutlineRhs = [] {
        if constexpr (requires { KernelPolicy<H>::kOutlineRhs; }) return KernelPolicy<H>::kOutlineRhs;
        else return false;
    }();
#endif
#ifdef ODEGPU_POLICY_BOOK_SHARED
    static constexpr bool kBookInShared = ODEGPU_POLICY_BOOK_SHARED;
#else
    static constexpr bool kBookInShared = [] {
        if constexpr (requires { KernelPolicy<H>::kBookInShared; }) return KernelPolicy<H>::kBookInShared;
        else return false; // specialisations written before the flag existed
    }();
#endif
    // the time-term cache (rk_step, TimeTermCache): time-split models with
    // straight-line stages, unless the policy declines it
    static constexpr bool kCacheTimeTerms = [] {
#ifdef ODEGPU_POLICY_CACHE_TT
        if constexpr (true) return ODEGPU_POLICY_CACHE_TT && kTimeTerms<H> > 0 && !kRolledStages;
        else
#endif
        if constexpr (requires { KernelPolicy<H>::kCacheTimeTerms; })
            return KernelPolicy<H>::kCacheTimeTerms && kTimeTerms<H> > 0 && !kRolledStages;
        else return kTimeTerms<H> > 0 && !kRolledStages;
    }();
    // cache slots: 1 (the end point: the next step's start — measured best,
    // cfg1 0.328 -> 0.314 ms, cfg3 13.0 -> 12.6 ms) or 2 (also a rejected
    // step's retry start)
    static constexpr int kTimeTermSlots = [] {
#ifdef ODEGPU_POLICY_TT_SLOTS
        if constexpr (true) return ODEGPU_POLICY_TT_SLOTS;
        else
#endif
        if constexpr (requires { KernelPolicy<H>::kTimeTermSlots; }) return KernelPolicy<H>::kTimeTermSlots;
        else return 1;
    }();
    static constexpr int kParamStride = kParamsInShared ? (H::kParamCount | 1) : 1;
    static constexpr int kParamRegs = kParamsInShared ? 1 : (H::kParamCount > 0 ? H::kParamCount : 1);
};

/// Everything a block keeps in shared memory, per policy (dynamic shared
/// memory: the Keller-Miksis layout exceeds the 48 KB static limit).
template <class H, Algorithm ALG, int BLOCK, class Pol = EffectivePolicy<H>>
struct SharedLayout {
    ColdState<H, Pol::kColdInShared ? BLOCK : 1, Pol::kCacheTimeTerms ? Pol::kTimeTermSlots : 0> cold;
    Bookkeeping<Pol::kBookInShared ? BLOCK : 1> book;
    Real params[Pol::kParamsInShared ? BLOCK * Pol::kParamStride : 1];
    Real k[Pol::kRolledStages ? (ALG == Algorithm::RK4 ? 3 : 5) * H::kSystemDim * BLOCK : 1];
};

/// Dynamic shared memory of one solve block.
template <class H, Algorithm ALG, int BLOCK>
constexpr std::size_t solve_smem_bytes() {
    return sizeof(SharedLayout<H, ALG, BLOCK>);
}

/// The ensemble loop. One instantiation per (model, algorithm): hooks are
/// inlined, widths are compile-time.
///
/// Each iteration: (1) PREPARE — lanes without a pending RK evaluation run
/// their bookkeeping (fetch + initialize a system, commit a detection step,
/// finalize + store, the secant update); (2) every lane evaluates one RK
/// step; (3) ABSORB — error control, and for the common outcome (rejected,
/// or accepted without an event detection) the whole of driver.hpp:146-227
/// inline in registers: landing, refresh of the event zones, accessories,
/// the next step's clipping — so a lane is ready for its next evaluation
/// without another trip through the state machine. Only detections, stops
/// and system ends go back through PREPARE.
///
/// STREAM: the streaming-pool instantiation (BatchArrays::gate); the
/// others carry none of its code.
template <class H, Algorithm ALG, int BLOCK, class Pol = EffectivePolicy<H>, bool LOG = false, bool STREAM = false>
__device__ __forceinline__ void solve_lanes(const H& m, const BatchArrays& b, const Controls& c) {
    constexpr int N = H::kSystemDim;
    constexpr int NP = H::kParamCount, NA = H::kAccessoryCount, E = H::kEventCount;
    constexpr int EE = E > 0 ? E : 1, A = NA > 0 ? NA : 1;
    constexpr bool kAdaptive = ALG == Algorithm::RKCK45;
    static_assert(N <= kMaxDim && E <= kMaxEvents, "model wider than the device controls");
    constexpr bool kFence = Pol::kColdInShared || Pol::kParamsInShared || Pol::kBookInShared;
    constexpr bool kCacheTT = Pol::kCacheTimeTerms;

    // cold state: a shared-memory column per thread, or a register record
    extern __shared__ __align__(16) unsigned char odegpu_dsmem[];
    auto& sh = *reinterpret_cast<SharedLayout<H, ALG, BLOCK, Pol>*>(odegpu_dsmem);
    ColdState<H, 1, Pol::kCacheTimeTerms ? Pol::kTimeTermSlots : 0> cs_regs;
    auto& cs = *[&] {
        if constexpr (Pol::kColdInShared) return &sh.cold;
        else return &cs_regs;
    }();
    const int tid = Pol::kColdInShared ? static_cast<int>(threadIdx.x) : 0;
    const TimeTermCache<std::remove_reference_t<decltype(cs)>, (kTimeTerms<H> > 0 ? kTimeTerms<H> : 1), kCacheTT,
                        Pol::kTimeTermSlots>
        ttc{
        cs, tid};
    if constexpr (kCacheTT) ttc.clear();
    Real* const sp = sh.params;
    // stage derivatives of the rolled stage loop (rk_step)
    Real* const kbuf = sh.k + (Pol::kRolledStages ? threadIdx.x : 0);
    const Index n = b.n;
    // STREAM: pending counts + the block's landed-granule watermark
    [[maybe_unused]] unsigned* const s_stream = stream_shared<STREAM, BLOCK>();
    // STREAM: a system's own t1 < t0 check (solve.hpp:159-161) as it is
    // taken up (true: not integrated, counted done and reported in bad[0]).
    // Run on the values the fetch loads anyway (late) where that is free;
    // before the loads (early) for models whose parameters live in shared
    // memory, whose register budget the late form overran (Keller-Miksis).
    constexpr bool kLateStreamChecks = !Pol::kParamsInShared;
    [[maybe_unused]] const auto stream_checks = [&](Real t0, Real t1, unsigned sys_) {
        if (t1 < t0) {
            atomicMin(b.gate.bad, static_cast<unsigned long long>(sys_));
            stream_release(b.gate, sys_);
            return true;
        }
        return false;
    };
    if constexpr (STREAM) {
        s_stream[threadIdx.x] = 0;
        if (threadIdx.x == 0) s_stream[BLOCK] = 0;
        __syncthreads();
    }
    Real preg[Pol::kParamRegs];
    Real* const prow = Pol::kParamsInShared ? sp + threadIdx.x * Pol::kParamStride : preg;

    const auto S = [](Real* a, int len) { return std::span<Real>(a, static_cast<std::size_t>(len)); };
    const auto CS = [](const Real* a, int len) { return std::span<const Real>(a, static_cast<std::size_t>(len)); };
#define ODEGPU_C(field) cs.field[tid]

    // ---- hot registers: the driver's loop variables (driver.hpp:96-107)
    Real t = 0, h_step = 0;
    Real y[N];
#pragma unroll
    for (int i = 0; i < N; ++i) y[i] = 0;
    bool clipped = false;
    // per-step bookkeeping (t1, smallest step, counters, event zones):
    // registers, or a shared-memory column when the policy parks it there
    // to free registers for the stages
    Bookkeeping<1> bk_regs;
    auto& bk = *[&] {
        if constexpr (Pol::kBookInShared) return &sh.book;
        else return &bk_regs;
    }();
    const int btid = Pol::kBookInShared ? static_cast<int>(threadIdx.x) : 0;
#define ODEGPU_B(field) bk.field[btid]
    int phase = kFetch;

    const auto load_acc = [&](Real (&a)[A]) {
#pragma unroll
        for (int i = 0; i < A; ++i) a[i] = ODEGPU_C(acc[i]);
    };
    const auto store_acc = [&](const Real (&a)[A]) {
#pragma unroll
        for (int i = 0; i < NA; ++i) ODEGPU_C(acc[i]) = a[i];
    };
    // driver.hpp:109-119: clip the next trial step onto t1; false when the
    // system is done (the lane goes to kFinish).
    // Written with selects, not branches: it runs after every trial step.
    // `live` is the loop condition t < t1 when the caller does not already
    // know it holds (after a rejection, or an accepted step that was not
    // clipped onto t1, it does).
    const auto setup_step = [&](bool check_live) {
        const Real t1 = ODEGPU_B(t1), h = ODEGPU_B(h);
        const bool live = !check_live || t < t1;
        clipped = t + h >= t1;
        const Real h_try = clipped ? t1 - t : h;
        const bool underflow = !(h_try > 0); // fp underflow of the remaining span: t = t1
        if (live && underflow) t = t1;
        h_step = h_try;
        phase = (live && !underflow) ? kReadyStep : kFinish;
    };
    // EventMachine::refresh (events.hpp:160-173) from post-action values.
    const auto refresh = [&](const Real (&fp)[EE]) {
        bool any_inside = false;
#pragma unroll
        for (int i = 0; i < E; ++i) {
            const int z = zone_of(fp[i], c.tolerance[i]);
            if (z == kZoneNone) continue; // non-finite: keep the previous arming
            ODEGPU_C(prev_value[i]) = fp[i];
            ODEGPU_B(zones) = with_zone(ODEGPU_B(zones), i, z);
            any_inside = any_inside || z == kZoneInside;
        }
        ODEGPU_B(steps_in_zone) = any_inside ? ODEGPU_B(steps_in_zone) + 1 : 0;
    };
    // refresh() given the zones of fp already computed.
    const auto refresh_zones = [&](const Real (&fp)[EE], const int (&zn)[EE]) {
        bool any_inside = false;
        int zones = ODEGPU_B(zones);
#pragma unroll
        for (int i = 0; i < E; ++i) {
            const bool keep = zn[i] == kZoneNone; // non-finite: keep the previous arming
            if (!keep) ODEGPU_C(prev_value[i]) = fp[i];
            zones = keep ? zones : with_zone(zones, i, zn[i]);
            any_inside = any_inside || zn[i] == kZoneInside;
        }
        ODEGPU_B(zones) = zones;
        ODEGPU_B(steps_in_zone) = any_inside ? ODEGPU_B(steps_in_zone) + 1 : 0;
    };
    // Ends a secant location (driver.hpp:157-164).
    const auto end_secant = [&]() {
        if (!ODEGPU_C(s_conv)) ++ODEGPU_C(n_secf);
        const bool rel = ODEGPU_C(b_th) < ODEGPU_C(h_try);
        ODEGPU_C(relocated) = rel;
        const Real tl = (ODEGPU_C(clipped) && !rel) ? ODEGPU_B(t1) : t + ODEGPU_C(b_th);
        ODEGPU_C(t_land) = tl;
        Real yl[N], f[EE];
#pragma unroll
        for (int i = 0; i < N; ++i) yl[i] = ODEGPU_C(y_land[i]);
        m.event_values(tl, CS(yl, N), CS(prow, NP), S(f, E));
#pragma unroll
        for (int i = 0; i < E; ++i) ODEGPU_C(f_land[i]) = f[i];
        phase = kCommit;
    };

    // Appends the detection records of a commit (BatchArrays::log_*): the
    // events in `mask`, classified against the zones before the commit,
    // counters and landed values from the cold state, y_land before and y
    // after the event action. Everything it reads lives in the cold state,
    // so the commit path keeps no extra registers for it.
    const auto log_detections = [&](const BatchArrays& bb, const Controls& cc, int zones_before, unsigned mask) {
        long long seq = static_cast<long long>(ODEGPU_C(n_det)) - __popc(mask); // n_det already counts them
#pragma unroll
        for (int i = 0; i < E; ++i) {
            if (!(mask >> i & 1u)) continue;
            const unsigned long long slot = atomicAdd(bb.log_count, 1ull);
            const long long q = seq++;
            if (slot >= static_cast<unsigned long long>(bb.log_capacity)) continue;
            const Index r = static_cast<Index>(slot);
            const Real v = ODEGPU_C(f_land[i]);
            const int prev = zone_at(zones_before, i);
            const int kn = classify_lut(prev, zone_of(v, cc.tolerance[i]), cc.kind_lut[i]);
            bb.log_system[r] = ODEGPU_C(sys);
            bb.log_event[r] = i;
            // SteppedAcross, EnteredFromAbove, EnteredFromBelow (events.hpp:31); a
            // forced (located, no longer classified) detection is SteppedAcross
            bb.log_kind[r] = kn == kKindEntered ? (prev == kZoneAbove ? 1 : 2) : 0;
            bb.log_in_zone[r] = isfinite(v) && fabs(v) <= cc.tolerance[i];
            bb.log_counter[r] = ODEGPU_C(counter[i]);
            bb.log_sequence[r] = q;
            bb.log_t[r] = t;
            bb.log_value[r] = v;
#pragma unroll
            for (int j = 0; j < N; ++j) {
                bb.log_y_pre[r + j * bb.log_capacity] = ODEGPU_C(y_land[j]);
                bb.log_y_post[r + j * bb.log_capacity] = y[j];
            }
        }
    };

    // One secant iteration's pre-step exits (events.hpp:214-219): the next
    // re-step length (kReadySecant), or the end of the location (kCommit).
    const auto secant_step = [&]() {
        if (ODEGPU_C(s_it) > kMaxSecantIterations) {
            end_secant();
            return;
        }
        const Real th_cur = ODEGPU_C(th_cur), f_cur = ODEGPU_C(f_cur);
        const Real denom = f_cur - ODEGPU_C(f_prev);
        if (denom == 0) {
            end_secant();
            return;
        }
        Real theta = th_cur - f_cur * (th_cur - ODEGPU_C(th_prev)) / denom;
        if (!isfinite(theta)) {
            end_secant();
            return;
        }
        const Real h_try = ODEGPU_C(h_try);
        theta = sclamp(theta, h_try * 1e-12, h_try); // th_min (events.hpp:209)
        if (theta == th_cur) {
            end_secant();
            return;
        }
        h_step = theta;
        phase = kReadySecant;
    };
#if ODEGPU_SECANT_INLINE
#define ODEGPU_SECANT_NEXT() secant_step()
#else
#define ODEGPU_SECANT_NEXT() (phase = kSecant)
#endif

    ODEGPU_C(lane_trial_steps) = 0ull;
    ODEGPU_C(lane_max_ratio) = 0.0;
    ODEGPU_C(lane_outside) = 0u;
    ODEGPU_C(lane_not_advanced) = 0u;
    ODEGPU_C(lane_detections) = 0u;

    for (;;) {
        // ================= PREPARE: bring this lane to a pending RK evaluation
        while (phase < kDone) {
            if (phase <= kRefetch) {
                // take up a system: the next one of the pool, or (fused
                // iterations) the same one again from the end point it just
                // stored — exactly what the next solve() would read
                Index sys;
                if (phase == kFetch) {
                    const Index j = fetch_system(b.work);
                    if constexpr (STREAM) { // the count of the system this lane finished last
                        const unsigned pend = s_stream[threadIdx.x];
                        if (pend) {
                            s_stream[threadIdx.x] = 0;
                            stream_release(b.gate, pend - 1);
                        }
                    }
                    if (j >= b.count) {
                        phase = kDone;
                        break;
                    }
                    sys = b.order ? static_cast<Index>(__ldg(b.order + j)) : j;
                    if constexpr (STREAM) { // streaming pool: the system's granule must have landed
                        if (!stream_wait(b.gate, s_stream + BLOCK, static_cast<unsigned>(sys))) {
                            stream_release(b.gate, static_cast<unsigned>(sys));
                            continue;
                        }
                        if constexpr (!kLateStreamChecks) {
                            if (stream_checks(b.td[sys], b.td[sys + n], static_cast<unsigned>(sys))) continue;
                        }
                    }
                    // solve.hpp:98 (never in a streaming run: it resets every outcome first)
                    if (b.reason[sys] == static_cast<std::uint8_t>(StopReason::NonFiniteAbort)) continue;
                    ODEGPU_C(it_left) = static_cast<unsigned short>(b.iterations);
                } else {
                    sys = static_cast<Index>(ODEGPU_C(sys));
                }
                ODEGPU_C(sys) = static_cast<unsigned>(sys);
                if constexpr (kCacheTT) ttc.clear(); // new parameters
                Real td[2] = {b.td[sys], b.td[sys + n]};
#pragma unroll
                for (int i = 0; i < N; ++i) y[i] = b.state[sys + i * n];
#pragma unroll
                for (int i = 0; i < NP; ++i) prow[i] = __ldg(b.params + sys + i * n);
                Real acc[A];
#pragma unroll
                for (int i = 0; i < NA; ++i) acc[i] = b.acc[sys + i * n];
                if constexpr (STREAM && kLateStreamChecks)
                    if (phase == kFetch && stream_checks(td[0], td[1], static_cast<unsigned>(sys))) continue;
                ODEGPU_B(n_acc) = ODEGPU_B(n_rej) = 0u;
                ODEGPU_C(acc_hi) = ODEGPU_C(rej_hi) = 0u;
                ODEGPU_C(n_det) = ODEGPU_C(n_secf) = 0ull;
                ODEGPU_C(n_resteps) = 0;
                ODEGPU_B(smallest) = __longlong_as_double(0x7ff0000000000000LL); // +inf
                ODEGPU_C(reason) = static_cast<std::uint8_t>(StopReason::ReachedEndTime);
                // driver.hpp:96-107
                m.initialize(td[0], S(td, 2), S(y, N), CS(prow, NP), S(acc, NA));
                ODEGPU_C(td[0]) = td[0];
                ODEGPU_C(td[1]) = td[1];
                store_acc(acc);
                t = td[0];
                ODEGPU_B(t1) = td[1];
                if constexpr (E > 0) { // EventMachine::init (events.hpp:93-101)
                    Real f0[EE];
                    m.event_values(t, CS(y, N), CS(prow, NP), S(f0, E));
                    ODEGPU_B(zones) = 0;
#pragma unroll
                    for (int i = 0; i < E; ++i) {
                        ODEGPU_C(prev_value[i]) = f0[i];
                        ODEGPU_B(zones) = with_zone(ODEGPU_B(zones), i, zone_of(f0[i], c.tolerance[i]));
                        ODEGPU_C(counter[i]) = 0;
                    }
                    ODEGPU_B(steps_in_zone) = 0;
                }
                ODEGPU_B(h) = kAdaptive ? sclamp(c.initial_time_step, c.min_step, c.max_step) : c.initial_time_step;
                phase = kSetup;
            }
            if (phase == kSetup) {
                setup_step(true);
                continue;
            }
            if (phase == kCommit) {
                // an accepted step with a detection: driver.hpp:170-227
                const Real tl = ODEGPU_C(t_land);
                if (tl <= t) {
                    ODEGPU_C(reason) = static_cast<std::uint8_t>(StopReason::NonFiniteAbort);
                    phase = kFinish;
                    continue;
                }
                const Real advanced = tl - t;
#pragma unroll
                for (int i = 0; i < N; ++i) y[i] = ODEGPU_C(y_land[i]);
                t = tl;
                if (++ODEGPU_B(n_acc) == 0u) ++ODEGPU_C(acc_hi);
                ODEGPU_B(smallest) = smin(ODEGPU_B(smallest), advanced);
                bool event_stop = false;
                Real acc[A];
                load_acc(acc);
                if constexpr (E > 0) {
                    const int located = ODEGPU_C(located);
                    bool det[EE];
                    long long cnt[EE];
#pragma unroll
                    for (int i = 0; i < E; ++i) { // EventMachine::commit, events.hpp:134-156
                        const int kind = classify_lut(zone_at(ODEGPU_B(zones), i),
                                                      zone_of(ODEGPU_C(f_land[i]), c.tolerance[i]), c.kind_lut[i]);
                        det[i] = kind != kKindNone || i == located;
                        cnt[i] = ODEGPU_C(counter[i]) + (det[i] ? 1 : 0);
                        ODEGPU_C(counter[i]) = cnt[i];
                        if (det[i]) {
                            ++ODEGPU_C(n_det);
                            ++ODEGPU_C(lane_detections);
                            // what the scans' detection observer records
                            // (src/scan.cpp:51-61): |F|/tol and in-zone
                            const Real v = ODEGPU_C(f_land[i]);
                            const bool fin = isfinite(v);
                            const Real ratio = fin ? fabs(v) / c.tolerance[i] : __longlong_as_double(0x7ff0000000000000LL);
                            if (!(fin && fabs(v) <= c.tolerance[i])) ++ODEGPU_C(lane_outside);
                            ODEGPU_C(lane_max_ratio) = smax(ODEGPU_C(lane_max_ratio), ratio);
                        }
                    }
                    // the zones the detections were classified against (refresh()
                    // re-arms them below): the detection log's kinds
                    const int zones_before = ODEGPU_B(zones);
                    Real f_post[EE];
                    if (located >= 0) {
#pragma unroll
                        for (int i = 0; i < E; ++i)
                            if (i == located) m.event_action(i, cnt[i], t, S(y, N), CS(prow, NP));
                        m.event_values(t, CS(y, N), CS(prow, NP), S(f_post, E));
                    } else {
#pragma unroll
                        for (int i = 0; i < E; ++i) f_post[i] = ODEGPU_C(f_land[i]);
                    }
                    refresh(f_post);
#pragma unroll
                    for (int i = 0; i < E; ++i)
                        if (det[i]) m.event_accessory(i, cnt[i], t, CS(y, N), CS(prow, NP), S(acc, NA));
                    if constexpr (LOG) { // the records, in event order (driver.hpp:204-206)
                        unsigned mask = 0;
#pragma unroll
                        for (int i = 0; i < E; ++i) mask |= det[i] ? 1u << i : 0u;
                        log_detections(b, c, zones_before, mask);
                    }
#pragma unroll
                    for (int i = 0; i < E; ++i)
                        if (det[i] && c.stop_condition[i] != 0 && cnt[i] >= c.stop_condition[i]) event_stop = true;
                }
                m.ordinary_accessory(t, CS(y, N), CS(prow, NP), S(acc, NA));
                store_acc(acc);
                if (event_stop) {
                    ODEGPU_C(reason) = static_cast<std::uint8_t>(StopReason::EventStop);
                    phase = kFinish;
                } else if (E > 0 && ODEGPU_B(steps_in_zone) >= c.max_steps_in_zone) {
                    ODEGPU_C(reason) = static_cast<std::uint8_t>(StopReason::EquilibriumStop);
                    phase = kFinish;
                } else {
                    if (kAdaptive && !ODEGPU_C(relocated)) ODEGPU_B(h) = ODEGPU_C(h_next);
                    setup_step(true);
                }
                continue;
            }
            if (phase == kFinish) {
                // driver.hpp:231-233, then scatter_system (batch.cpp:32-40)
                Real td[2] = {ODEGPU_C(td[0]), ODEGPU_C(td[1])};
                Real acc[A];
                load_acc(acc);
                m.finalize(t, S(td, 2), S(y, N), CS(prow, NP), S(acc, NA));
                const Index sys = static_cast<Index>(ODEGPU_C(sys));
                // scan start-time check (src/scan.cpp:296-298): b.td still
                // holds t0 as fetched
                if (ODEGPU_C(reason) != static_cast<std::uint8_t>(StopReason::NonFiniteAbort) &&
                    !(td[0] > b.td[sys]))
                    ++ODEGPU_C(lane_not_advanced);
                b.td[sys] = td[0];
                b.td[sys + n] = td[1];
#pragma unroll
                for (int i = 0; i < N; ++i) b.state[sys + i * n] = y[i];
#pragma unroll
                for (int i = 0; i < NA; ++i) b.acc[sys + i * n] = acc[i];
                b.final_t[sys] = t;
                b.reason[sys] = ODEGPU_C(reason);
                const Index acc64 = static_cast<Index>((static_cast<unsigned long long>(ODEGPU_C(acc_hi)) << 32) |
                                                       ODEGPU_B(n_acc));
                const Index rej64 = static_cast<Index>((static_cast<unsigned long long>(ODEGPU_C(rej_hi)) << 32) |
                                                       ODEGPU_B(n_rej));
                b.accepted[sys] = acc64;
                b.rejected[sys] = rej64;
                b.detections[sys] = static_cast<Index>(ODEGPU_C(n_det));
                b.secant_failures[sys] = static_cast<Index>(ODEGPU_C(n_secf));
                if (b.cost) { // fetch-order key (saturates: only the order of long systems is at stake)
                    const unsigned long long c64 = static_cast<unsigned long long>(acc64) +
                                                   static_cast<unsigned long long>(rej64) + ODEGPU_C(n_resteps);
                    b.cost[sys] = c64 > 0xffffffffull ? 0xffffffffu : static_cast<unsigned>(c64);
                }
                b.smallest_step[sys] = ODEGPU_B(smallest);
                ODEGPU_C(lane_trial_steps) += static_cast<unsigned long long>(acc64) + static_cast<unsigned long long>(rej64);
                // fused iterations: solve the same system again unless it
                // aborted (a NonFiniteAbort outcome is sticky, solve.hpp:98)
                const unsigned short left = static_cast<unsigned short>(ODEGPU_C(it_left) - 1);
                ODEGPU_C(it_left) = left;
                phase = (left > 0 && ODEGPU_C(reason) != static_cast<std::uint8_t>(StopReason::NonFiniteAbort))
                            ? kRefetch
                            : kFetch;
                if constexpr (STREAM) // the system's last solve of this launch
                    if (phase == kFetch) {
                        stream_finish(b.gate, static_cast<unsigned>(sys), t, ODEGPU_C(reason), acc64, rej64,
                                      static_cast<Index>(ODEGPU_C(n_det)), static_cast<Index>(ODEGPU_C(n_secf)),
                                      ODEGPU_B(smallest));
                        s_stream[threadIdx.x] = static_cast<unsigned>(sys) + 1u; // counted at the next fetch
                    }
                continue;
            }
            if (phase == kSecant) {
                secant_step();
                continue;
            }
        }
        // Warp-uniform exit: every lane stays resident until its whole warp
        // is done, and the vote re-converges the warp, so the RK stages below
        // always run once per iteration for all lanes (finished lanes compute
        // on stale state and ignore the result).
        if (__all_sync(0xffffffffu, phase == kDone)) {
            if (b.trial_steps) {
                unsigned long long st = ODEGPU_C(lane_trial_steps);
                for (int o = 16; o > 0; o >>= 1) st += __shfl_xor_sync(0xffffffffu, st, o);
                if ((threadIdx.x & 31) == 0 && st) atomicAdd(b.trial_steps, st);
            }
            if (b.tally) { // warp-reduced scan tally, one atomic per counter and warp
                unsigned outside = ODEGPU_C(lane_outside), not_adv = ODEGPU_C(lane_not_advanced);
                unsigned dets = ODEGPU_C(lane_detections);
                Real mr = ODEGPU_C(lane_max_ratio);
                for (int o = 16; o > 0; o >>= 1) {
                    outside += __shfl_xor_sync(0xffffffffu, outside, o);
                    not_adv += __shfl_xor_sync(0xffffffffu, not_adv, o);
                    dets += __shfl_xor_sync(0xffffffffu, dets, o);
                    mr = smax(mr, __shfl_xor_sync(0xffffffffu, mr, o));
                }
                if ((threadIdx.x & 31) == 0) {
                    // detections counted where they happen (the reference's
                    // detection observer): a sticky-aborted system's stale
                    // outcome record is not re-counted in later iterations
                    if (dets) atomicAdd(b.tally + kTallyDetections, static_cast<unsigned long long>(dets));
                    if (outside) atomicAdd(b.tally + kTallyOutsideZone, static_cast<unsigned long long>(outside));
                    if (not_adv) atomicAdd(b.tally + kTallyStartNotAdvanced, static_cast<unsigned long long>(not_adv));
                    if (mr > 0) atomicMax(b.tally + kTallyMaxRatio, static_cast<unsigned long long>(__double_as_longlong(mr)));
                }
            }
            break;
        }

        // ================= the shared Runge-Kutta evaluation
        if constexpr (kFence) cold_fence();
        Real yn[N], err[N];
        const bool nonfinite =
            rk_step<H, ALG, Pol::kRolledStages, BLOCK, Pol::kOutlineRhs>(m, t, h_step, y, prow, yn, err, kbuf, ttc);
        if constexpr (kFence) cold_fence();

        // ================= ABSORB
        if (phase == kReadyStep) {
            const Real h_try = h_step;
            Real h_next = ODEGPU_B(h);
            if constexpr (!kAdaptive) {
                if (nonfinite) { // driver.hpp:124-128
                    ODEGPU_C(reason) = static_cast<std::uint8_t>(StopReason::NonFiniteAbort);
                    phase = kFinish;
                    continue;
                }
            } else {
                // error_ratio (steppers.hpp:154-163) + control_step (176-198).
                // (The branch-free Divisor form of these quotients measured
                // slower here: 2.27 vs 2.16 ms on cfg2.)
                Real ratio = 0.0;
#pragma unroll
                for (int i = 0; i < N; ++i) {
                    // std::max(|y|, |yn|) selected on the raw values and made
                    // absolute in the DFMA operand (no DADDs materialising |y|)
                    const Real big = fabs((fabs(y[i]) < fabs(yn[i])) ? yn[i] : y[i]);
                    const Real scale = c.abs_tol[i] + c.rel_tol[i] * big;
                    ratio = smax(ratio, err[i] / scale);
                }
                bool accepted;
                if (nonfinite) {
                    if (h_try <= c.min_step) {
                        ODEGPU_C(reason) = static_cast<std::uint8_t>(StopReason::NonFiniteAbort);
                        phase = kFinish;
                        continue;
                    }
                    accepted = false;
                    h_next = smax(h_try * c.step_shrink_limit, c.min_step);
                } else {
                    accepted = ratio <= 1.0;
                    Real factor = 0.9 * dmath::controller_pow(ratio); // std::pow(ratio, -0.2)
                    factor = sclamp(factor, c.step_shrink_limit, c.step_grow_limit);
                    h_next = sclamp(h_try * factor, c.min_step, c.max_step);
                    if (!accepted && h_try <= c.min_step) {
                        accepted = true;
                        h_next = c.min_step;
                    }
                }
                if (!accepted) { // driver.hpp:136-140; t < t1 still holds
                    if (++ODEGPU_B(n_rej) == 0u) ++ODEGPU_C(rej_hi);
                    ODEGPU_B(h) = h_next;
                    setup_step(false);
                    continue;
                }
            }
            // accepted: driver.hpp:146-168
            const Real tl = clipped ? ODEGPU_B(t1) : t + h_try;
            if constexpr (E > 0) {
                Real f[EE];
                m.event_values(tl, CS(yn, N), CS(prow, NP), S(f, E));
                // EventMachine::peek (events.hpp:111-125): highest index wins
                int located = -1, kind = kKindNone;
                int zn[EE]; // the landed zones, also what refresh() stores
#pragma unroll
                for (int i = 0; i < E; ++i) zn[i] = zone_of(f[i], c.tolerance[i]);
#pragma unroll
                for (int i = 0; i < E; ++i) { // ascending: the highest index wins
                    const int k = classify_lut(zone_at(ODEGPU_B(zones), i), zn[i], c.kind_lut[i]);
                    located = k != kKindNone ? i : located;
                    kind = k != kKindNone ? k : kind;
                }
                if (located >= 0) { // detection: the slow path through PREPARE
                    ODEGPU_C(t_land) = tl;
#pragma unroll
                    for (int i = 0; i < N; ++i) ODEGPU_C(y_land[i]) = yn[i];
#pragma unroll
                    for (int i = 0; i < E; ++i) ODEGPU_C(f_land[i]) = f[i];
                    ODEGPU_C(h_next) = h_next;
                    ODEGPU_C(located) = located;
                    ODEGPU_C(relocated) = false;
                    phase = kCommit;
                    if (kind == kKindAcross) {
                        // start locate_secant (events.hpp:207-212); y_land holds y(h)
                        ODEGPU_C(h_try) = h_try;
                        ODEGPU_C(clipped) = clipped;
                        ODEGPU_C(s_idx) = located;
                        ODEGPU_C(s_it) = 1;
                        ODEGPU_C(s_conv) = false;
                        ODEGPU_C(th_prev) = 0;
                        ODEGPU_C(th_cur) = h_try;
                        Real fp = 0, fc = 0;
#pragma unroll
                        for (int i = 0; i < E; ++i)
                            if (i == located) {
                                fp = ODEGPU_C(prev_value[i]);
                                fc = f[i];
                            }
                        ODEGPU_C(f_prev) = fp;
                        ODEGPU_C(f_cur) = fc;
                        ODEGPU_C(b_th) = h_try;
                        ODEGPU_C(b_f) = fc;
                        ODEGPU_SECANT_NEXT();
                    }
                    continue;
                }
                if (tl <= t) { // driver.hpp:170-173
                    ODEGPU_C(reason) = static_cast<std::uint8_t>(StopReason::NonFiniteAbort);
                    phase = kFinish;
                    continue;
                }
                refresh_zones(f, zn); // no detection: commit records nothing, f_post = f_landed
            } else {
                if (tl <= t) {
                    ODEGPU_C(reason) = static_cast<std::uint8_t>(StopReason::NonFiniteAbort);
                    phase = kFinish;
                    continue;
                }
            }
            ODEGPU_B(smallest) = smin(ODEGPU_B(smallest), tl - t);
#pragma unroll
            for (int i = 0; i < N; ++i) y[i] = yn[i];
            t = tl;
            if (++ODEGPU_B(n_acc) == 0u) ++ODEGPU_C(acc_hi);
            if constexpr (kHasOrdinaryAccessory<H>) {
                Real acc[A];
                load_acc(acc);
                m.ordinary_accessory(t, CS(y, N), CS(prow, NP), S(acc, NA));
                store_acc(acc);
            }
            if (E > 0 && ODEGPU_B(steps_in_zone) >= c.max_steps_in_zone) {
                ODEGPU_C(reason) = static_cast<std::uint8_t>(StopReason::EquilibriumStop);
                phase = kFinish;
                continue;
            }
            ODEGPU_B(h) = h_next;
            // landed on t1 exactly when clipped (driver.hpp:146): the loop ends
            if (clipped) phase = kFinish;
            else setup_step(false);
        } else if (phase == kReadySecant) { // one secant iteration's step is in (events.hpp:222-240)
            if constexpr (E > 0) {
                if (ODEGPU_C(n_resteps) != 0xffff) ++ODEGPU_C(n_resteps);
                Real fs[EE];
                m.event_values(t + h_step, CS(yn, N), CS(prow, NP), S(fs, E));
                const int s_idx = ODEGPU_C(s_idx);
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
                if (fabs(f) < fabs(ODEGPU_C(b_f))) {
                    ODEGPU_C(b_th) = h_step;
                    ODEGPU_C(b_f) = f;
#pragma unroll
                    for (int i = 0; i < N; ++i) ODEGPU_C(y_land[i]) = yn[i];
                }
                if (fabs(f) <= tol) {
                    ODEGPU_C(s_conv) = true;
                    end_secant();
                    continue;
                }
                ODEGPU_C(th_prev) = ODEGPU_C(th_cur);
                ODEGPU_C(f_prev) = ODEGPU_C(f_cur);
                ODEGPU_C(th_cur) = h_step;
                ODEGPU_C(f_cur) = f;
                ++ODEGPU_C(s_it);
                ODEGPU_SECANT_NEXT();
            }
        }
    }
#undef ODEGPU_C
#undef ODEGPU_B
#undef ODEGPU_SECANT_NEXT
}

/// A model whose hooks have a CertifiedTrig twin (include/odegpu/trig.hpp).
template <class H>
concept TrigCertifiable = requires(Real t, const Real* p, Index stride) {
    typename H::certified_hooks;
    { H::trig_argument_bound(t, t, p, stride) } -> std::convertible_to<Real>;
} && std::is_empty_v<typename H::certified_hooks> && H::kSystemDim == H::certified_hooks::kSystemDim &&
    H::kParamCount == H::certified_hooks::kParamCount && H::kEventCount == H::certified_hooks::kEventCount &&
    H::kAccessoryCount == H::certified_hooks::kAccessoryCount;

/// Trig certificate of a batch: flags[1] stays 0 only if every system that
/// will be integrated has all trig arguments below kTrigCertifiedLimit over
/// its time domain (a non-finite bound fails). Reads td plus the parameters
/// the bound needs; launched right before the solve kernel.
template <class H>
__global__ void trig_certificate_kernel(BatchArrays b, unsigned long long* flags) {
    for (Index i = blockIdx.x * static_cast<Index>(blockDim.x) + threadIdx.x; i < b.count;
         i += static_cast<Index>(gridDim.x) * blockDim.x) {
        if (b.reason[i] == static_cast<std::uint8_t>(StopReason::NonFiniteAbort)) continue; // skipped by solve
        const Real bound = H::trig_argument_bound(b.td[i], b.td[i + b.n], b.params + i, b.n);
        if (!(bound < kTrigCertifiedLimit)) flags[1] = 1;
    }
}

/// The solve kernel. flags[0] is the result of the t1 < t0 check queued
/// before it: when a system failed it, nothing is integrated (the reference
/// throws before solving, solve.hpp:159-161). flags[1] == 0 is the batch's
/// trig certificate: the model's certified_hooks instantiation (no range
/// branch in its trig) runs instead of the general one; both share one
/// shared-memory layout and policy.
///
/// LOG: the instantiation that also records every detection (BatchArrays
/// log_*, the reference's on_detection observer), launched only while a
/// batch has a detection log — like the reference's `observing` branch
/// (driver.hpp:186-206) it costs nothing when nobody observes.
///
/// STREAM: the streaming-pool instantiation (odegpu_pipeline STREAMING):
/// lanes wait on the granule gate, check t1 < t0 per system, and write
/// packed records and per-group counts. A streaming run takes the general
/// trig path (flags[1] != 0): the certificate needs every system before the
/// launch, and a second launch for systems a certified pass would have to
/// leave out could wait behind the copy-out stream's value waits.
template <class H, Algorithm ALG, int BLOCK, int MIN_BLOCKS, bool LOG = false, bool STREAM = false>
__global__ void __launch_bounds__(BLOCK, MIN_BLOCKS)
    guarded_solve_kernel(H model, BatchArrays b, Controls c, const unsigned long long* flags) {
    if (flags[0] != ~0ull) return;
    dmath::init_shared_tables();
    if constexpr (TrigCertifiable<H> && !STREAM) {
        if (flags[1] == 0) {
            solve_lanes<typename H::certified_hooks, ALG, BLOCK, EffectivePolicy<H>, LOG, STREAM>(
                typename H::certified_hooks{}, b, c);
            return;
        }
    }
    solve_lanes<H, ALG, BLOCK, EffectivePolicy<H>, LOG, STREAM>(model, b, c);
}

/// Kernel controls from the C-ABI structs (materialised once per solve,
/// solve.hpp:153-155); the caller has validated them.
inline Controls controls_from(const odegpu_system_dims& sys, const odegpu_solver_config& cfg,
                              const odegpu_ode_controls& ode, const odegpu_event_controls* ev) {
    Controls c{};
    for (Index i = 0; i < sys.system_dim; ++i) {
        c.rel_tol[i] = ode.rel_tol[i];
        c.abs_tol[i] = ode.abs_tol[i];
    }
    c.max_step = ode.max_step;
    c.min_step = ode.min_step;
    c.step_grow_limit = ode.step_grow_limit;
    c.step_shrink_limit = ode.step_shrink_limit;
    c.initial_time_step = cfg.initial_time_step;
    c.max_steps_in_zone = ev ? ev->max_steps_in_zone : 50;
    for (Index i = 0; i < sys.event_count; ++i) {
        c.direction[i] = ev->direction[i];
        c.kind_lut[i] = kind_table(ev->direction[i]);
        c.tolerance[i] = ev->tolerance[i];
        c.stop_condition[i] = ev->stop_condition[i];
    }
    return c;
}

} // namespace odegpu::device

#endif
