// launch.cuh — instantiation and launch of the per-model solve kernels.
// Included by the model translation units (models_*.cu) only.
#pragma once

#include <atomic>

#include "internal.cuh"

namespace odegpu::detail {

using dev::guarded_solve_kernel;

/// Per-model launch policy: resident blocks of kBlock threads per SM that
/// __launch_bounds__ asks ptxas for (register cap 65536 / (kMinBlocks *
/// kBlock)). Chosen per model family from ncu runs;
/// ODEGPU_MIN_BLOCKS overrides it for tuning builds.
/// ODEGPU_MB(x): a model's chosen minimum resident blocks, unless a tuning
/// build forces one value for every model (-DODEGPU_MIN_BLOCKS).
#ifdef ODEGPU_MIN_BLOCKS
#define ODEGPU_MB(x) ODEGPU_MIN_BLOCKS
#else
#define ODEGPU_MB(x) (x)
#endif

constexpr int kMaxDevices = 64; // occupancy cache slots (per device ordinal)

template <class H>
struct LaunchPolicy {
    static constexpr int kBlock = detail::kBlock;
#ifdef ODEGPU_MIN_BLOCKS
    static constexpr int kMinBlocks = ODEGPU_MIN_BLOCKS;
#else
    static constexpr int kMinBlocks = 4;
#endif
};

template <class H, Algorithm ALG>
void launch_one(odegpu_batch* b, const H& hooks, const dev::Controls& c) {
    constexpr int kMin = LaunchPolicy<H>::kMinBlocks;
    constexpr int kBlock = [] {
#ifdef ODEGPU_BLOCK // tuning builds: one block size for every model
        return ODEGPU_BLOCK;
#else
        if constexpr (requires { LaunchPolicy<H>::kBlock; }) return LaunchPolicy<H>::kBlock;
        else return detail::kBlock;
#endif
    }();
    // the detection-log instantiation only for models with events, and only
    // while the batch has a log (odegpu_batch_set_detection_log); its own
    // launch bounds leave it one block per SM fewer (more registers for the
    // observer path instead of spills)
    const bool log = H::kEventCount > 0 && b->a.log_count != nullptr;
    // streaming pool (pipeline.cu): its own instantiation; the caller has set
    // both flags (general trig path), fetch in natural order
    const bool streaming = b->stream_mode != 0;
    auto kern = guarded_solve_kernel<H, ALG, kBlock, kMin, false, false>;
    if constexpr (H::kEventCount > 0)
        if (log) kern = guarded_solve_kernel<H, ALG, kBlock, (kMin > 1 ? kMin - 1 : 1), true, false>;
    // (one block per SM fewer, like the log: the streaming pass runs the
    // general trig path plus its gate, and stays spill-free)
    if (streaming) kern = guarded_solve_kernel<H, ALG, kBlock, (kMin > 1 ? kMin - 1 : 1), false, true>;
    const int variant = streaming ? 2 : log ? 1 : 0;
    constexpr std::size_t smem = dev::solve_smem_bytes<H, ALG, kBlock>();
    if constexpr (smem > 48 * 1024) // opt-in above the static limit (per device)
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    // resident blocks per SM, per instantiation and device: device threads of
    // odegpu_solve_pool_multi launch concurrently, and devices may differ
    static std::atomic<int> resident_of[3][kMaxDevices] = {};
    auto& cache = resident_of[variant];
    int resident = b->device >= 0 && b->device < kMaxDevices ? cache[b->device].load(std::memory_order_relaxed) : 0;
    if (resident <= 0) {
        int r = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&r, kern, kBlock, smem));
        resident = std::max(r, 1);
        if (b->device >= 0 && b->device < kMaxDevices) cache[b->device].store(resident, std::memory_order_relaxed);
    }
    const Index n = b->a.count;
    const Index persistent = Index(b->num_sms) * resident;
    const Index needed = (n + kBlock - 1) / kBlock;
    const int grid = static_cast<int>(std::max<Index>(1, std::min(needed, persistent)));
    if constexpr (dev::TrigCertifiable<H>) if (!streaming) {
        CK(cudaMemsetAsync(b->first_bad + 1, 0, sizeof(unsigned long long), b->stream));
        dev::trig_certificate_kernel<H><<<grid_for(b, b->a.count, 256), 256, 0, b->stream>>>(b->a, b->first_bad);
        CK(cudaGetLastError());
        ++b->launches;
    }
    CK(cudaMemsetAsync(b->a.work, 0, sizeof(unsigned long long), b->stream));
    // AUTO: longest-first for adaptive steppers of models whose policy asks
    // for it (a fixed step count per system gives nothing to order)
    constexpr bool kPolicyCost = [] {
        if constexpr (requires { LaunchPolicy<H>::kCostOrder; })
            return LaunchPolicy<H>::kCostOrder && ALG == Algorithm::RKCK45;
        else return false;
    }();
    const bool cost = !streaming && (b->order_mode == ODEGPU_FETCH_COST ||
                                     (b->order_mode == ODEGPU_FETCH_AUTO && kPolicyCost));
    b->a.order = (!streaming && cost && b->order_count == n) ? b->order : nullptr;
    b->a.cost = (cost && b->build_order) ? b->cost : nullptr; // null until the first order build allocates it
    // fused iterations: the systems of this launch are solved `fused` times
    // in a row (hooks.hpp kFusableIterations; one solve otherwise)
    // (not with a detection log: its records belong to one solve)
    const Index fused = kFusableIterations<H> && !b->a.log_count
                            ? std::max<Index>(1, std::min<Index>(b->fuse_request, 65535))
                            : 1;
    if (b->a.log_count) CK(cudaMemsetAsync(b->a.log_count, 0, sizeof(unsigned long long), b->stream));
    b->a.iterations = static_cast<int>(fused);
    b->fused_done = fused;
    b->fuse_request = 1;
    b->a.trial_steps = b->trial_steps;
    CK(cudaEventRecord(b->ev_start, b->stream));
    kern<<<grid, kBlock, smem, b->stream>>>(hooks, b->a, c, b->first_bad);
    CK(cudaGetLastError());
    CK(cudaEventRecord(b->ev_stop, b->stream));
    b->a.iterations = 1;
    b->a.order = nullptr;
    const bool have_cost = b->a.cost != nullptr;
    b->a.cost = nullptr;
    b->timed = true;
    ++b->launches;
    if (cost && b->build_order) build_cost_order(b, have_cost); // for the next solve of this batch
}

template <class H>
void launch_alg(odegpu_batch* b, const H& hooks, int algorithm, const dev::Controls& c) {
    if (algorithm == ODEGPU_RK4)
        launch_one<H, Algorithm::RK4>(b, hooks, c);
    else
        launch_one<H, Algorithm::RKCK45>(b, hooks, c);
}

template <class H>
void set_dims(odegpu_system_dims* d, bool* keeps_time_domain = nullptr, bool* fusable = nullptr) {
    *d = odegpu_system_dims{H::kSystemDim, H::kParamCount, H::kEventCount, H::kAccessoryCount};
    if (keeps_time_domain) *keeps_time_domain = kKeepsTimeDomain<H>;
    if (fusable) *fusable = kFusableIterations<H>;
}

} // namespace odegpu::detail
