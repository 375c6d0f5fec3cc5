// internal.cuh — shared internals of libodegpu: error plumbing, the batch
// object behind the C ABI, and the host-side helpers the ABI, the model
// translation units and the pool pipeline share. Not installed.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <new>
#include <stdexcept>
#include <string>

#include "odegpu.h"
#include "odegpu/device/solver.cuh"

namespace odegpu::detail {

namespace dev = odegpu::device;

/// Message of the last failing ABI call on this thread (odegpu_last_error).
inline thread_local std::string g_err;

struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void throw_invalid(const std::string& m) { throw Error(ODEGPU_ERR_INVALID_ARGUMENT, m); }
[[noreturn]] inline void throw_range(const std::string& m) { throw Error(ODEGPU_ERR_OUT_OF_RANGE, m); }
[[noreturn]] inline void throw_unsupported(const std::string& m) { throw Error(ODEGPU_ERR_UNSUPPORTED, m); }

inline void check_cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw Error(ODEGPU_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define CK(x) ::odegpu::detail::check_cuda((x), #x)

/// Runs f, mapping exceptions to ABI return codes and g_err.
template <typename F>
int guarded(F&& f) {
    try {
        f();
        g_err.clear();
        return ODEGPU_OK;
    } catch (const Error& e) {
        g_err = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        g_err = "host allocation failed";
        return ODEGPU_ERR_CUDA;
    } catch (const std::exception& e) {
        g_err = e.what();
        return ODEGPU_ERR_CUDA;
    }
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int d) {
        cudaGetDevice(&prev);
        if (prev != d) CK(cudaSetDevice(d));
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

constexpr int kBlock = 128; // threads per block of the solve kernels

} // namespace odegpu::detail

/// The batch behind the C ABI (SolverBatch, batch.hpp:17-67): one device
/// allocation holding the SoA arrays, a stream, validation scratch.
struct odegpu_batch {
    odegpu_batch_dims dims{};
    int device = 0;
    cudaStream_t stream = nullptr;     // stream all work is ordered on
    cudaStream_t own_stream = nullptr; // the batch's private stream
    odegpu::device::BatchArrays a{};
    unsigned long long* first_bad = nullptr; // solve-time validation result (device)
    unsigned long long* host_flag = nullptr;  // pinned mirror of first_bad
    unsigned long long* diag = nullptr;       // device tally (9 counters)
    cudaEvent_t ev_start = nullptr, ev_stop = nullptr; // brackets the last solve kernel
    bool timed = false;
    int num_sms = 0;
    int64_t launches = 0;
    void* block = nullptr;     // single device allocation backing every array
    void* out_stage = nullptr; // lazily allocated pinned OutcomeStage for reads
    // fetch order (odegpu_batch_set_fetch_order): a permutation of
    // [0, order_count) built after each COST-mode solve (build_cost_order)
    int32_t order_mode = ODEGPU_FETCH_AUTO;
    odegpu::Index order_count = -1;
    void* order_block = nullptr; // order + sort keys/values + CUB scratch
    unsigned* order = nullptr;
    unsigned* cost = nullptr; // per-system RK evaluations of the last COST-mode solve (BatchArrays::cost)
    bool build_order = true; // false: the next solve's order would go unused (pipeline, last iteration)
    // fused iterations (solver.cuh BatchArrays::iterations): how many solves
    // the next launch may run per system, and how many the last one ran
    // (1 for models whose finalize could invalidate the time domain)
    odegpu::Index fuse_request = 1;
    odegpu::Index fused_done = 1;
    unsigned long long* trial_steps = nullptr; // device: trial steps integrated since the last reset
    void* log_block = nullptr; // detection log (odegpu_batch_set_detection_log), BatchArrays::log_*
    // streaming pool run (pipeline.cu): nonzero = the launch is the
    // streaming pass (STREAM instantiation, natural fetch order; the caller
    // has set both flags, so no certificate pre-pass)
    int stream_mode = 0;
};

namespace odegpu::detail {

inline void check_batch(const odegpu_batch* b) {
    if (!b) throw_invalid("null batch");
}

inline int grid_for(const odegpu_batch* b, Index work, int block) {
    const Index g = (work + block - 1) / block;
    return static_cast<int>(std::max<Index>(1, std::min<Index>(g, Index(b->num_sms) * 8)));
}

// ---- kernels.cu: small kernels, launched on the batch stream
void launch_reset_outcomes(odegpu_batch* b, Index start, Index count);
void launch_reset_rows(odegpu_batch* b, const Index* d_idx, Index count);
void launch_scatter_rows(odegpu_batch* b, Real* dst, const Index* d_idx, const Real* staged, Index count,
                         Index components);
void enqueue_time_check(odegpu_batch* b); // solve.hpp:159-161 on [0, a.count)
void launch_diagnostics(odegpu_batch* b);
// longest-first fetch order from the last solve's RK evaluations (its cost
// array when the kernel wrote it, else accepted + rejected steps)
void build_cost_order(odegpu_batch* b, bool have_cost);
void launch_tally(odegpu_batch* b, unsigned long long* tally, bool chunk_end); // scan outcome tally
double run_dfma_peak(int blocks, int threads, int iters, double* seconds);

// ---- model translation units: widths and kernel dispatch per model family
bool family_dims_duffing(const odegpu_model& m, odegpu_system_dims* d, bool* keeps = nullptr, bool* fusable = nullptr);
bool family_dims_keller_miksis(const odegpu_model& m, odegpu_system_dims* d, bool* keeps = nullptr, bool* fusable = nullptr);
bool family_dims_valve(const odegpu_model& m, odegpu_system_dims* d, bool* keeps = nullptr, bool* fusable = nullptr);
bool family_dims_fakes(const odegpu_model& m, odegpu_system_dims* d, bool* keeps = nullptr, bool* fusable = nullptr);
bool family_launch_duffing(odegpu_batch* b, const odegpu_model& m, int alg, const dev::Controls& c);
bool family_launch_keller_miksis(odegpu_batch* b, const odegpu_model& m, int alg, const dev::Controls& c);
bool family_launch_valve(odegpu_batch* b, const odegpu_model& m, int alg, const dev::Controls& c);
bool family_launch_fakes(odegpu_batch* b, const odegpu_model& m, int alg, const dev::Controls& c);

// ---- api.cu
odegpu_system_dims dims_of(const odegpu_model& m);
// whether a solve of the model leaves time domains unchanged (hooks.hpp kKeepsTimeDomain)
bool keeps_time_domain(const odegpu_model& m);
// whether solve_iteratively may fuse the model's iterations into one launch (hooks.hpp kFusableIterations)
bool fusable_iterations(const odegpu_model& m);
void launch_model(odegpu_batch* b, const odegpu_model& m, int algorithm, const dev::Controls& c);
dev::Controls prepare_solve(const odegpu_batch_dims& d, const odegpu_model* m, const odegpu_solver_config* cfg,
                            const odegpu_ode_controls* ode, const odegpu_event_controls* ev);
dev::Controls validate_solve(const odegpu_batch_dims& d, const odegpu_system_dims& sys,
                             const odegpu_solver_config* cfg, const odegpu_ode_controls* ode,
                             const odegpu_event_controls* ev);
void raise_if_bad(odegpu_batch* b); // syncs the batch stream
void copy_h2d_strided(Real* dst, Index dst_stride, Index dst_start, const double* src, Index src_stride,
                      Index src_start, Index count, Index components, cudaStream_t s);
void copy_d2h_strided(double* dst, Index dst_stride, Index dst_start, const Real* src, Index src_stride,
                      Index src_start, Index count, Index components, cudaStream_t s);
odegpu_batch* batch_create(const odegpu_batch_dims& dims, int device); // throws
Index components_of(const odegpu_batch_dims& d, int32_t property);
Real* property_ptr(odegpu_batch* b, int32_t property);
const double* pool_ptr(const odegpu_pool_view* p, int32_t property);
bool wants(int32_t mode, int32_t which);
void check_dims_agree(const odegpu_batch_dims& b, const odegpu_pool_dims& p);

/// Page-locked host blocks through a process-wide cache (pipeline.cu): a
/// freed block is kept for reuse (pinning is slow) up to a size limit.
void* host_alloc(size_t bytes);
void host_free(void* p);

/// Pinned staging for the SoA outcome fields of `cap` systems.
struct OutcomeStage {
    double* final_t = nullptr;
    double* smallest = nullptr;
    Index* accepted = nullptr;
    Index* rejected = nullptr;
    Index* detections = nullptr;
    Index* secant_failures = nullptr;
    std::uint8_t* reason = nullptr;
    void* block = nullptr;
    void allocate(Index cap);
    void release();
    /// async D2H of batch outcomes [start, start+count) into slots [0, count)
    void fetch(const odegpu_batch* b, Index start, Index count, cudaStream_t s);
    /// AoS records (odensemble::SystemOutcome layout) from slots [0, count)
    void pack(odegpu_outcome* out, Index count) const;
};
void download_outcomes(odegpu_batch* b, Index start, Index count, odegpu_outcome* host); // synchronous
void release_batch_stage(odegpu_batch* b);

} // namespace odegpu::detail

namespace odegpu::detail {
void run_math_check(int fn, Index n, const double* x, const double* y, double* mine, double* ref);
} // namespace odegpu::detail
