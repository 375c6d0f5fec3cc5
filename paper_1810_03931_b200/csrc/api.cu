// api.cu — implementation of the C ABI (include/odegpu.h): device-resident
// SoA batches, pool<->batch copies, validation with the reference's messages,
// and dispatch of the per-model sm_100a solve kernels.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <mutex>
#include <new>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "odegpu.h"
#include "odegpu/device/solver.cuh"
#include "odegpu/models/duffing.hpp"
#include "odegpu/models/keller_miksis.hpp"
#include "odegpu/models/valve.hpp"
#include "test_fakes.cuh"

using namespace odegpu;
namespace dev = odegpu::device;

static_assert(sizeof(odegpu_outcome) == 56, "odegpu_outcome must match odensemble::SystemOutcome");

namespace {

thread_local std::string g_err;

struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] void throw_invalid(const std::string& m) { throw Error(ODEGPU_ERR_INVALID_ARGUMENT, m); }
[[noreturn]] void throw_range(const std::string& m) { throw Error(ODEGPU_ERR_OUT_OF_RANGE, m); }

void check_cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw Error(ODEGPU_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define CK(x) check_cuda((x), #x)

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

// ------------------------------------------------------------ device kernels

__global__ void reset_outcomes_kernel(dev::BatchArrays b, Index start, Index count) {
    for (Index i = blockIdx.x * static_cast<Index>(blockDim.x) + threadIdx.x; i < count;
         i += static_cast<Index>(gridDim.x) * blockDim.x) {
        const Index s = start + i;
        b.final_t[s] = 0.0;
        b.reason[s] = 0;
        b.accepted[s] = 0;
        b.rejected[s] = 0;
        b.detections[s] = 0;
        b.secant_failures[s] = 0;
        b.smallest_step[s] = __longlong_as_double(0x7ff0000000000000LL);
    }
}

// solve.hpp:159-161: lowest index with t1 < t0 (or n if none).
__global__ void check_time_domains_kernel(const Real* td, Index n, unsigned long long* first_bad) {
    for (Index i = blockIdx.x * static_cast<Index>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<Index>(gridDim.x) * blockDim.x)
        if (td[i + n] < td[i]) atomicMin(first_bad, static_cast<unsigned long long>(i));
}

// batch[dst[j] + c*nb] = staged[j + c*count] for every component c.
__global__ void scatter_rows_kernel(Real* dst, Index nb, const Index* idx, const Real* staged, Index count,
                                    Index components) {
    const Index total = count * components;
    for (Index k = blockIdx.x * static_cast<Index>(blockDim.x) + threadIdx.x; k < total;
         k += static_cast<Index>(gridDim.x) * blockDim.x) {
        const Index c = k / count, j = k - c * count;
        dst[idx[j] + c * nb] = staged[k];
    }
}

__global__ void reset_rows_kernel(dev::BatchArrays b, const Index* idx, Index count) {
    for (Index j = blockIdx.x * static_cast<Index>(blockDim.x) + threadIdx.x; j < count;
         j += static_cast<Index>(gridDim.x) * blockDim.x) {
        const Index s = idx[j];
        b.final_t[s] = 0.0;
        b.reason[s] = 0;
        b.accepted[s] = 0;
        b.rejected[s] = 0;
        b.detections[s] = 0;
        b.secant_failures[s] = 0;
        b.smallest_step[s] = __longlong_as_double(0x7ff0000000000000LL);
    }
}

// The skip flag: when the time-domain check found a bad system the solve
// kernel must not touch anything (the reference throws before solving).
template <class H, Algorithm ALG, int BLOCK, int MINB>
__global__ void __launch_bounds__(BLOCK, MINB)
    guarded_solve_kernel(H model, dev::BatchArrays b, dev::Controls c, const unsigned long long* first_bad) {
    if (*first_bad != ~0ull) return;
    dev::solve_lanes<H, ALG>(model, b, c);
}

// Outcome tally (ScanDiagnostics::tally_iteration, src/scan.cpp:63-68).
// acc[0..3] = sums, acc[4..7] = reason counts, acc[8] = max trial steps.
__global__ void diagnostics_kernel(dev::BatchArrays b, unsigned long long* acc) {
    unsigned long long s_acc = 0, s_rej = 0, s_det = 0, s_sf = 0, r[4] = {0, 0, 0, 0}, mx = 0;
    for (Index i = blockIdx.x * static_cast<Index>(blockDim.x) + threadIdx.x; i < b.n;
         i += static_cast<Index>(gridDim.x) * blockDim.x) {
        s_acc += b.accepted[i];
        s_rej += b.rejected[i];
        s_det += b.detections[i];
        s_sf += b.secant_failures[i];
        const unsigned rs = b.reason[i] & 3u;
        r[0] += rs == 0;
        r[1] += rs == 1;
        r[2] += rs == 2;
        r[3] += rs == 3;
        const unsigned long long tr = static_cast<unsigned long long>(b.accepted[i] + b.rejected[i]);
        mx = tr > mx ? tr : mx;
    }
    for (int o = 16; o > 0; o >>= 1) {
        s_acc += __shfl_down_sync(0xffffffffu, s_acc, o);
        s_rej += __shfl_down_sync(0xffffffffu, s_rej, o);
        s_det += __shfl_down_sync(0xffffffffu, s_det, o);
        s_sf += __shfl_down_sync(0xffffffffu, s_sf, o);
        for (int k = 0; k < 4; ++k) r[k] += __shfl_down_sync(0xffffffffu, r[k], o);
        const unsigned long long m2 = __shfl_down_sync(0xffffffffu, mx, o);
        mx = m2 > mx ? m2 : mx;
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(acc + 0, s_acc);
        atomicAdd(acc + 1, s_rej);
        atomicAdd(acc + 2, s_det);
        atomicAdd(acc + 3, s_sf);
        for (int k = 0; k < 4; ++k) atomicAdd(acc + 4 + k, r[k]);
        atomicMax(acc + 8, mx);
    }
}

// FP64 peak microbenchmark: 8 independent DFMA chains per thread.
__global__ void dfma_peak_kernel(double* out, int iters, double seed) {
    double a0 = seed + threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6,
           a7 = a0 + 7;
    const double b = 0.999999, c = 1e-7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            a0 = fma(a0, b, c);
            a1 = fma(a1, b, c);
            a2 = fma(a2, b, c);
            a3 = fma(a3, b, c);
            a4 = fma(a4, b, c);
            a5 = fma(a5, b, c);
            a6 = fma(a6, b, c);
            a7 = fma(a7, b, c);
        }
    }
    const double s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
    if (s == 12345.678) out[0] = s; // keep the chains alive
}

} // namespace

// ------------------------------------------------------------ the batch

struct odegpu_batch {
    odegpu_batch_dims dims{};
    int device = 0;
    cudaStream_t stream = nullptr;     // stream all work is ordered on
    cudaStream_t own_stream = nullptr; // the batch's private stream
    dev::BatchArrays a{};
    unsigned long long* first_bad = nullptr; // solve-time validation result
    unsigned long long* host_flag = nullptr;  // pinned mirror of first_bad
    unsigned long long* diag = nullptr;       // device tally (9 counters)
    cudaEvent_t ev_start = nullptr, ev_stop = nullptr; // brackets the last solve kernel
    bool timed = false;
    int num_sms = 0;
    int64_t launches = 0;
    void* block = nullptr; // single device allocation backing every array
};

namespace {

size_t align_up(size_t v) { return (v + 255) & ~size_t(255); }

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

void check_batch(const odegpu_batch* b) {
    if (!b) throw_invalid("null batch");
}

Index components_of(const odegpu_batch_dims& d, int32_t property) {
    switch (property) {
    case ODEGPU_PROP_TIME_DOMAIN: return 2;
    case ODEGPU_PROP_STATE: return d.system_dim;
    case ODEGPU_PROP_PARAMETERS: return d.param_count;
    case ODEGPU_PROP_ACCESSORIES: return d.accessory_count;
    default: throw_invalid("unknown property");
    }
}

Real* property_ptr(odegpu_batch* b, int32_t property) {
    switch (property) {
    case ODEGPU_PROP_TIME_DOMAIN: return b->a.td;
    case ODEGPU_PROP_STATE: return b->a.state;
    case ODEGPU_PROP_PARAMETERS: return const_cast<Real*>(b->a.params);
    case ODEGPU_PROP_ACCESSORIES: return b->a.acc;
    default: throw_invalid("unknown property");
    }
}

const double* pool_ptr(const odegpu_pool_view* p, int32_t property) {
    switch (property) {
    case ODEGPU_PROP_TIME_DOMAIN: return p->time_domain;
    case ODEGPU_PROP_STATE: return p->state;
    case ODEGPU_PROP_PARAMETERS: return p->parameters;
    case ODEGPU_PROP_ACCESSORIES: return p->accessories;
    default: return nullptr;
    }
}

bool wants(int32_t mode, int32_t which) { return mode == which || mode == ODEGPU_COPY_ALL; } // batch.cpp:74

void check_dims_agree(const odegpu_batch_dims& b, const odegpu_pool_dims& p) { // batch.cpp:48-52
    if (b.system_dim != p.system_dim || b.param_count != p.param_count || b.accessory_count != p.accessory_count)
        throw_invalid("copy: batch and pool disagree on per-system dimensions");
}

int grid_for(const odegpu_batch* b, Index work, int block) {
    const Index g = (work + block - 1) / block;
    return static_cast<int>(std::max<Index>(1, std::min<Index>(g, Index(b->num_sms) * 8)));
}

// ------------------------------------------------------------ model table

odegpu_system_dims dims_of(const odegpu_model& m) {
    auto d = [](auto h) {
        using H = decltype(h);
        return odegpu_system_dims{H::kSystemDim, H::kParamCount, H::kEventCount, H::kAccessoryCount};
    };
    switch (m.id) {
    case ODEGPU_MODEL_DUFFING: return d(models::DuffingHooks{});
    case ODEGPU_MODEL_DUFFING_MAX_ACCESSORY: return d(models::DuffingMaxAccessoryHooks{});
    case ODEGPU_MODEL_DUFFING_MAX_EVENT: return d(models::DuffingMaxEventHooks{});
    case ODEGPU_MODEL_DUFFING_MAXMIN: return d(models::DuffingMaxMinHooks{});
    case ODEGPU_MODEL_KELLER_MIKSIS: return d(models::KellerMiksisHooks{});
    case ODEGPU_MODEL_BUBBLE_COLLAPSE: return d(models::BubbleCollapseHooks{});
    case ODEGPU_MODEL_VALVE: return d(models::ValveHooks{});
    case ODEGPU_MODEL_DUFFING_LYAPUNOV: return d(models::DuffingLyapunovHooks{});
    case ODEGPU_MODEL_CONSTANT: return d(fakes::ConstantHooks{});
    case ODEGPU_MODEL_CUBIC_TIME: return d(fakes::CubicTimeHooks{});
    case ODEGPU_MODEL_EXPONENTIAL: return d(fakes::ExponentialHooks{});
    case ODEGPU_MODEL_UNIT_SLOPE: return d(fakes::UnitSlopeHooks{});
    case ODEGPU_MODEL_COUNTING: return d(fakes::CountingHooks{});
    case ODEGPU_MODEL_RAMP: return d(fakes::RampHooks{});
    case ODEGPU_MODEL_DECAY: return d(fakes::DecayHooks{});
    case ODEGPU_MODEL_SEAT_CONTACT: return d(fakes::SeatContactHooks{});
    case ODEGPU_MODEL_HARMONIC: return d(fakes::HarmonicHooks{});
    case ODEGPU_MODEL_BLOWUP: return d(fakes::BlowUpHooks{});
    default: throw Error(ODEGPU_ERR_UNSUPPORTED, "unknown model id " + std::to_string(m.id));
    }
}

constexpr int kBlock = 128;

template <class H, Algorithm ALG>
void launch_one(odegpu_batch* b, const H& hooks, const dev::Controls& c) {
    auto kern = guarded_solve_kernel<H, ALG, kBlock, 1>;
    static int resident = -1; // per instantiation: resident blocks per SM
    if (resident < 0) {
        int r = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&r, kern, kBlock, 0));
        resident = std::max(r, 1);
    }
    const Index n = b->dims.batch_capacity;
    const Index persistent = Index(b->num_sms) * resident;
    const Index needed = (n + kBlock - 1) / kBlock;
    const int grid = static_cast<int>(std::max<Index>(1, std::min(needed, persistent)));
    CK(cudaMemsetAsync(b->a.work, 0, sizeof(unsigned long long), b->stream));
    CK(cudaEventRecord(b->ev_start, b->stream));
    kern<<<grid, kBlock, 0, b->stream>>>(hooks, b->a, c, b->first_bad);
    CK(cudaGetLastError());
    CK(cudaEventRecord(b->ev_stop, b->stream));
    b->timed = true;
    ++b->launches;
}

template <class H>
void launch_alg(odegpu_batch* b, const H& hooks, int algorithm, const dev::Controls& c) {
    if (algorithm == ODEGPU_RK4)
        launch_one<H, Algorithm::RK4>(b, hooks, c);
    else
        launch_one<H, Algorithm::RKCK45>(b, hooks, c);
}

void launch_model(odegpu_batch* b, const odegpu_model& m, int algorithm, const dev::Controls& c) {
    const double* k = m.consts;
    switch (m.id) {
    case ODEGPU_MODEL_DUFFING: return launch_alg(b, models::DuffingHooks{}, algorithm, c);
    case ODEGPU_MODEL_DUFFING_MAX_ACCESSORY: return launch_alg(b, models::DuffingMaxAccessoryHooks{}, algorithm, c);
    case ODEGPU_MODEL_DUFFING_MAX_EVENT: return launch_alg(b, models::DuffingMaxEventHooks{}, algorithm, c);
    case ODEGPU_MODEL_DUFFING_MAXMIN: return launch_alg(b, models::DuffingMaxMinHooks{}, algorithm, c);
    case ODEGPU_MODEL_KELLER_MIKSIS: return launch_alg(b, models::KellerMiksisHooks{}, algorithm, c);
    case ODEGPU_MODEL_BUBBLE_COLLAPSE: return launch_alg(b, models::BubbleCollapseHooks{}, algorithm, c);
    case ODEGPU_MODEL_VALVE: return launch_alg(b, models::ValveHooks{}, algorithm, c);
    case ODEGPU_MODEL_DUFFING_LYAPUNOV: return launch_alg(b, models::DuffingLyapunovHooks{}, algorithm, c);
    case ODEGPU_MODEL_CONSTANT: {
        fakes::ConstantHooks h;
        h.value = k[0];
        return launch_alg(b, h, algorithm, c);
    }
    case ODEGPU_MODEL_CUBIC_TIME: return launch_alg(b, fakes::CubicTimeHooks{}, algorithm, c);
    case ODEGPU_MODEL_EXPONENTIAL: return launch_alg(b, fakes::ExponentialHooks{}, algorithm, c);
    case ODEGPU_MODEL_UNIT_SLOPE: return launch_alg(b, fakes::UnitSlopeHooks{}, algorithm, c);
    case ODEGPU_MODEL_COUNTING: return launch_alg(b, fakes::CountingHooks{}, algorithm, c);
    case ODEGPU_MODEL_RAMP: {
        fakes::RampHooks h;
        h.slope = k[0];
        h.level = k[1];
        return launch_alg(b, h, algorithm, c);
    }
    case ODEGPU_MODEL_DECAY: return launch_alg(b, fakes::DecayHooks{}, algorithm, c);
    case ODEGPU_MODEL_SEAT_CONTACT: return launch_alg(b, fakes::SeatContactHooks{}, algorithm, c);
    case ODEGPU_MODEL_HARMONIC: return launch_alg(b, fakes::HarmonicHooks{}, algorithm, c);
    case ODEGPU_MODEL_BLOWUP: return launch_alg(b, fakes::BlowUpHooks{}, algorithm, c);
    default: throw Error(ODEGPU_ERR_UNSUPPORTED, "unknown model id " + std::to_string(m.id));
    }
}

// solve.hpp:145-157: validation that needs no device data, plus control
// materialisation into the kernel-parameter struct.
dev::Controls prepare_solve(odegpu_batch* b, const odegpu_model* m, const odegpu_solver_config* cfg,
                            const odegpu_ode_controls* ode, const odegpu_event_controls* ev) {
    check_batch(b);
    if (!m || !cfg || !ode) throw_invalid("solve: null argument");
    const odegpu_system_dims sys = dims_of(*m);
    const auto& d = b->dims;
    if (sys.system_dim != d.system_dim || sys.param_count != d.param_count || sys.event_count != d.event_count ||
        sys.accessory_count != d.accessory_count)
        throw_invalid("solve: definition and batch dimensions disagree");
    if (cfg->initial_time_step <= 0) throw_invalid("solve: initial_time_step must be > 0");
    if (cfg->tile_size < 1) throw_invalid("solve: tile_size must be >= 1");
    if (cfg->algorithm != ODEGPU_RK4 && cfg->algorithm != ODEGPU_RKCK45) throw_invalid("solve: unknown algorithm");
    if (cfg->algorithm != ODEGPU_RK4 && cfg->initial_time_step > ode->max_step)
        throw_invalid("solve: initial_time_step exceeds max_step");
    if (sys.system_dim > dev::kMaxDim || sys.event_count > dev::kMaxEvents)
        throw Error(ODEGPU_ERR_UNSUPPORTED, "solve: model wider than the device controls");
    if (!ode->rel_tol || !ode->abs_tol) throw_invalid("solve: null tolerance arrays");
    if (sys.event_count > 0 && (!ev || !ev->direction || !ev->tolerance || !ev->stop_condition))
        throw_invalid("solve: event controls missing");

    dev::Controls c{};
    for (Index i = 0; i < sys.system_dim; ++i) {
        c.rel_tol[i] = ode->rel_tol[i];
        c.abs_tol[i] = ode->abs_tol[i];
    }
    c.max_step = ode->max_step;
    c.min_step = ode->min_step;
    c.step_grow_limit = ode->step_grow_limit;
    c.step_shrink_limit = ode->step_shrink_limit;
    c.initial_time_step = cfg->initial_time_step;
    c.max_steps_in_zone = ev ? ev->max_steps_in_zone : 50;
    for (Index i = 0; i < sys.event_count; ++i) {
        c.direction[i] = ev->direction[i];
        c.tolerance[i] = ev->tolerance[i];
        c.stop_condition[i] = ev->stop_condition[i];
    }
    return c;
}

// Device-side t1 < t0 check (solve.hpp:159-161) into b->first_bad.
void enqueue_time_check(odegpu_batch* b) {
    const Index n = b->dims.batch_capacity;
    CK(cudaMemsetAsync(b->first_bad, 0xff, sizeof(unsigned long long), b->stream));
    check_time_domains_kernel<<<grid_for(b, n, 256), 256, 0, b->stream>>>(b->a.td, n, b->first_bad);
    CK(cudaGetLastError());
    ++b->launches;
}

void raise_if_bad(odegpu_batch* b) {
    CK(cudaMemcpyAsync(b->host_flag, b->first_bad, sizeof(unsigned long long), cudaMemcpyDeviceToHost, b->stream));
    CK(cudaStreamSynchronize(b->stream));
    if (*b->host_flag != ~0ull)
        throw_invalid("solve: system " + std::to_string(static_cast<long long>(*b->host_flag)) + " has t1 < t0");
}

void copy_h2d_strided(Real* dst, Index dst_stride, Index dst_start, const double* src, Index src_stride,
                      Index src_start, Index count, Index components, cudaStream_t s) {
    if (count == 0 || components == 0) return;
    // one 2D copy: `components` rows of `count` doubles (batch.cpp:55-63)
    CK(cudaMemcpy2DAsync(dst + dst_start, size_t(dst_stride) * sizeof(Real), src + src_start,
                         size_t(src_stride) * sizeof(double), size_t(count) * sizeof(Real), size_t(components),
                         cudaMemcpyHostToDevice, s));
}

} // namespace

// ============================================================ C ABI

extern "C" {

int odegpu_abi_version(void) { return ODEGPU_ABI_VERSION; }

const char* odegpu_last_error(void) { return g_err.c_str(); }

int odegpu_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

int odegpu_model_dims(const odegpu_model* model, odegpu_system_dims* out) {
    return guarded([&] {
        if (!model || !out) throw_invalid("null argument");
        *out = dims_of(*model);
    });
}

int odegpu_batch_create(const odegpu_batch_dims* dims, int device, odegpu_batch** out) {
    return guarded([&] {
        if (!dims || !out) throw_invalid("null argument");
        *out = nullptr;
        // BatchDims::validate (pool.hpp:67-73)
        if (dims->batch_capacity < 1) throw_invalid("BatchDims: batch_capacity must be >= 1");
        if (dims->system_dim < 1) throw_invalid("BatchDims: system_dim must be >= 1");
        if (dims->param_count < 0) throw_invalid("BatchDims: param_count must be >= 0");
        if (dims->event_count < 0) throw_invalid("BatchDims: event_count must be >= 0");
        if (dims->accessory_count < 0) throw_invalid("BatchDims: accessory_count must be >= 0");
        DeviceGuard g(device);
        auto* b = new odegpu_batch;
        b->dims = *dims;
        b->device = device;
        try {
            CK(cudaDeviceGetAttribute(&b->num_sms, cudaDevAttrMultiProcessorCount, device));
            CK(cudaStreamCreateWithFlags(&b->own_stream, cudaStreamNonBlocking));
            b->stream = b->own_stream;
            const size_t n = size_t(dims->batch_capacity);
            const size_t sizes[] = {
                2 * n * 8,                                 // td
                size_t(dims->system_dim) * n * 8,          // state
                size_t(dims->param_count) * n * 8,         // params
                size_t(dims->accessory_count) * n * 8,     // acc
                n * 8,                                     // final_t
                n,                                         // reason
                n * 8, n * 8, n * 8, n * 8,                // counters
                n * 8,                                     // smallest
                8, 8, 128};                                // work, first_bad, diag
            size_t total = 0;
            for (size_t s : sizes) total += align_up(s);
            CK(cudaMalloc(&b->block, total));
            CK(cudaMemsetAsync(b->block, 0, total, b->stream));
            char* p = static_cast<char*>(b->block);
            void* ptrs[14];
            for (int i = 0; i < 14; ++i) {
                ptrs[i] = p;
                p += align_up(sizes[i]);
            }
            b->a.td = static_cast<Real*>(ptrs[0]);
            b->a.state = static_cast<Real*>(ptrs[1]);
            b->a.params = static_cast<Real*>(ptrs[2]);
            b->a.acc = static_cast<Real*>(ptrs[3]);
            b->a.final_t = static_cast<Real*>(ptrs[4]);
            b->a.reason = static_cast<std::uint8_t*>(ptrs[5]);
            b->a.accepted = static_cast<Index*>(ptrs[6]);
            b->a.rejected = static_cast<Index*>(ptrs[7]);
            b->a.detections = static_cast<Index*>(ptrs[8]);
            b->a.secant_failures = static_cast<Index*>(ptrs[9]);
            b->a.smallest_step = static_cast<Real*>(ptrs[10]);
            b->a.work = static_cast<unsigned long long*>(ptrs[11]);
            b->first_bad = static_cast<unsigned long long*>(ptrs[12]);
            b->diag = static_cast<unsigned long long*>(ptrs[13]);
            CK(cudaEventCreate(&b->ev_start));
            CK(cudaEventCreate(&b->ev_stop));
            b->a.n = dims->batch_capacity;
            CK(cudaMallocHost(&b->host_flag, sizeof(unsigned long long)));
            reset_outcomes_kernel<<<grid_for(b, dims->batch_capacity, 256), 256, 0, b->stream>>>(
                b->a, 0, dims->batch_capacity);
            CK(cudaGetLastError());
            CK(cudaStreamSynchronize(b->stream));
        } catch (...) {
            odegpu_batch_destroy(b);
            throw;
        }
        *out = b;
    });
}

void odegpu_batch_destroy(odegpu_batch* b) {
    if (!b) return;
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(b->device);
    if (b->stream) cudaStreamSynchronize(b->stream);
    if (b->block) cudaFree(b->block);
    if (b->host_flag) cudaFreeHost(b->host_flag);
    if (b->ev_start) cudaEventDestroy(b->ev_start);
    if (b->ev_stop) cudaEventDestroy(b->ev_stop);
    if (b->own_stream) cudaStreamDestroy(b->own_stream);
    if (prev >= 0) cudaSetDevice(prev);
    delete b;
}

int odegpu_batch_dims_get(const odegpu_batch* b, odegpu_batch_dims* out) {
    return guarded([&] {
        check_batch(b);
        if (!out) throw_invalid("null argument");
        *out = b->dims;
    });
}

int odegpu_batch_set_stream(odegpu_batch* b, void* stream) {
    return guarded([&] {
        check_batch(b);
        DeviceGuard g(b->device);
        CK(cudaStreamSynchronize(b->stream));
        b->stream = stream ? static_cast<cudaStream_t>(stream) : b->own_stream;
    });
}

int odegpu_linear_set(odegpu_batch* b, const odegpu_pool_view* pool, const odegpu_linear_copy_spec* spec) {
    return guarded([&] {
        check_batch(b);
        if (!pool || !spec) throw_invalid("null argument");
        // batch.cpp:79-85
        check_dims_agree(b->dims, pool->dims);
        if (spec->element_count < 0 || spec->start_in_batch < 0 || spec->start_in_pool < 0)
            throw_range("linear_set: negative index or count");
        if (spec->start_in_batch + spec->element_count > b->dims.batch_capacity)
            throw_range("linear_set: range exceeds batch capacity");
        if (spec->start_in_pool + spec->element_count > pool->dims.problem_size)
            throw_range("linear_set: range exceeds pool size");
        if (spec->copy_mode < ODEGPU_COPY_TIME_DOMAIN || spec->copy_mode > ODEGPU_COPY_ALL)
            throw_invalid("linear_set: unknown copy mode");
        DeviceGuard g(b->device);
        const Index nb = b->dims.batch_capacity, np = pool->dims.problem_size, n = spec->element_count;
        for (int32_t prop = ODEGPU_PROP_TIME_DOMAIN; prop <= ODEGPU_PROP_ACCESSORIES; ++prop) {
            if (!wants(spec->copy_mode, prop)) continue; // CopyMode value == property value
            const Index comps = components_of(b->dims, prop);
            if (comps == 0 || n == 0) continue;
            const double* src = pool_ptr(pool, prop);
            if (!src) throw_invalid("linear_set: pool array missing");
            copy_h2d_strided(property_ptr(b, prop), nb, spec->start_in_batch, src, np, spec->start_in_pool, n,
                             comps, b->stream);
        }
        if (n > 0) { // batch.cpp:102-103
            reset_outcomes_kernel<<<grid_for(b, n, 256), 256, 0, b->stream>>>(b->a, spec->start_in_batch, n);
            CK(cudaGetLastError());
        }
        CK(cudaStreamSynchronize(b->stream)); // host pool buffers may be reused on return
    });
}

int odegpu_random_set(odegpu_batch* b, const odegpu_pool_view* pool, const odegpu_index* ib,
                      const odegpu_index* ip, odegpu_index count, int32_t copy_mode) {
    return guarded([&] {
        check_batch(b);
        if (!pool) throw_invalid("null argument");
        check_dims_agree(b->dims, pool->dims); // batch.cpp:107-117
        if (count < 0) throw_invalid("random_set: index lists differ in length");
        if (count > 0 && (!ib || !ip)) throw_invalid("random_set: index lists differ in length");
        std::unordered_set<Index> seen;
        for (Index j = 0; j < count; ++j) {
            const Index i = ib[j];
            if (i < 0 || i >= b->dims.batch_capacity) throw_range("random_set: batch index out of range");
            if (!seen.insert(i).second) throw_invalid("random_set: duplicate batch index " + std::to_string(i));
        }
        for (Index j = 0; j < count; ++j)
            if (ip[j] < 0 || ip[j] >= pool->dims.problem_size) throw_range("random_set: pool index out of range");
        if (copy_mode < ODEGPU_COPY_TIME_DOMAIN || copy_mode > ODEGPU_COPY_ALL)
            throw_invalid("random_set: unknown copy mode");
        if (count == 0) return;
        DeviceGuard g(b->device);
        const Index nb = b->dims.batch_capacity, np = pool->dims.problem_size;
        // gather on the host into one staging block, one H2D, scatter on device
        Index total_comps = 0;
        for (int32_t prop = 0; prop <= ODEGPU_PROP_ACCESSORIES; ++prop)
            if (wants(copy_mode, prop)) total_comps += components_of(b->dims, prop);
        std::vector<double> staged(size_t(total_comps * count));
        Index* d_idx = nullptr;
        double* d_staged = nullptr;
        CK(cudaMallocAsync(reinterpret_cast<void**>(&d_idx), size_t(count) * sizeof(Index), b->stream));
        CK(cudaMallocAsync(reinterpret_cast<void**>(&d_staged), staged.size() * sizeof(double) + 8, b->stream));
        CK(cudaMemcpyAsync(d_idx, ib, size_t(count) * sizeof(Index), cudaMemcpyHostToDevice, b->stream));
        Index off = 0;
        for (int32_t prop = 0; prop <= ODEGPU_PROP_ACCESSORIES; ++prop) {
            if (!wants(copy_mode, prop)) continue;
            const Index comps = components_of(b->dims, prop);
            if (comps == 0) continue;
            const double* src = pool_ptr(pool, prop);
            if (!src) throw_invalid("random_set: pool array missing");
            for (Index c = 0; c < comps; ++c)
                for (Index j = 0; j < count; ++j) staged[size_t(off + c * count + j)] = src[ip[j] + c * np];
            off += comps * count;
        }
        CK(cudaMemcpyAsync(d_staged, staged.data(), staged.size() * sizeof(double), cudaMemcpyHostToDevice,
                           b->stream));
        off = 0;
        for (int32_t prop = 0; prop <= ODEGPU_PROP_ACCESSORIES; ++prop) {
            if (!wants(copy_mode, prop)) continue;
            const Index comps = components_of(b->dims, prop);
            if (comps == 0) continue;
            scatter_rows_kernel<<<grid_for(b, count * comps, 256), 256, 0, b->stream>>>(
                property_ptr(b, prop), nb, d_idx, d_staged + off, count, comps);
            CK(cudaGetLastError());
            off += comps * count;
        }
        reset_rows_kernel<<<grid_for(b, count, 256), 256, 0, b->stream>>>(b->a, d_idx, count); // batch.cpp:134
        CK(cudaGetLastError());
        CK(cudaFreeAsync(d_idx, b->stream));
        CK(cudaFreeAsync(d_staged, b->stream));
        CK(cudaStreamSynchronize(b->stream));
    });
}

int odegpu_batch_read_range(odegpu_batch* b, int32_t property, odegpu_index start, odegpu_index count,
                            double* host, odegpu_index host_stride) {
    return guarded([&] {
        check_batch(b);
        const Index comps = components_of(b->dims, property);
        if (start < 0 || count < 0 || start + count > b->dims.batch_capacity) throw_range("read: range out of bounds");
        if (host_stride < count) throw_invalid("read: host stride < count");
        if (comps == 0 || count == 0) return;
        if (!host) throw_invalid("null argument");
        DeviceGuard g(b->device);
        CK(cudaMemcpy2DAsync(host, size_t(host_stride) * 8, property_ptr(b, property) + start,
                             size_t(b->dims.batch_capacity) * 8, size_t(count) * 8, size_t(comps),
                             cudaMemcpyDeviceToHost, b->stream));
        CK(cudaStreamSynchronize(b->stream));
    });
}

int odegpu_batch_write_range(odegpu_batch* b, int32_t property, odegpu_index start, odegpu_index count,
                             const double* host, odegpu_index host_stride) {
    return guarded([&] {
        check_batch(b);
        const Index comps = components_of(b->dims, property);
        if (start < 0 || count < 0 || start + count > b->dims.batch_capacity)
            throw_range("write: range out of bounds");
        if (host_stride < count) throw_invalid("write: host stride < count");
        if (comps == 0 || count == 0) return;
        if (!host) throw_invalid("null argument");
        DeviceGuard g(b->device);
        copy_h2d_strided(property_ptr(b, property), b->dims.batch_capacity, start, host, host_stride, 0, count,
                         comps, b->stream);
        CK(cudaStreamSynchronize(b->stream));
    });
}

int odegpu_batch_read(odegpu_batch* b, int32_t property, double* host) {
    if (!b) return guarded([] { throw_invalid("null batch"); });
    return odegpu_batch_read_range(b, property, 0, b->dims.batch_capacity, host, b->dims.batch_capacity);
}

int odegpu_batch_write(odegpu_batch* b, int32_t property, const double* host) {
    if (!b) return guarded([] { throw_invalid("null batch"); });
    return odegpu_batch_write_range(b, property, 0, b->dims.batch_capacity, host, b->dims.batch_capacity);
}

int odegpu_batch_read_outcomes(odegpu_batch* b, odegpu_outcome* host) {
    return guarded([&] {
        check_batch(b);
        if (!host) throw_invalid("null argument");
        DeviceGuard g(b->device);
        const size_t n = size_t(b->dims.batch_capacity);
        std::vector<double> ft(n), ss(n);
        std::vector<Index> acc(n), rej(n), det(n), sf(n);
        std::vector<std::uint8_t> rs(n);
        CK(cudaMemcpyAsync(ft.data(), b->a.final_t, n * 8, cudaMemcpyDeviceToHost, b->stream));
        CK(cudaMemcpyAsync(rs.data(), b->a.reason, n, cudaMemcpyDeviceToHost, b->stream));
        CK(cudaMemcpyAsync(acc.data(), b->a.accepted, n * 8, cudaMemcpyDeviceToHost, b->stream));
        CK(cudaMemcpyAsync(rej.data(), b->a.rejected, n * 8, cudaMemcpyDeviceToHost, b->stream));
        CK(cudaMemcpyAsync(det.data(), b->a.detections, n * 8, cudaMemcpyDeviceToHost, b->stream));
        CK(cudaMemcpyAsync(sf.data(), b->a.secant_failures, n * 8, cudaMemcpyDeviceToHost, b->stream));
        CK(cudaMemcpyAsync(ss.data(), b->a.smallest_step, n * 8, cudaMemcpyDeviceToHost, b->stream));
        CK(cudaStreamSynchronize(b->stream));
        for (size_t i = 0; i < n; ++i) {
            odegpu_outcome o{};
            o.final_t = ft[i];
            o.reason = rs[i];
            o.accepted_steps = acc[i];
            o.rejected_steps = rej[i];
            o.event_detections = det[i];
            o.secant_failures = sf[i];
            o.smallest_step = ss[i];
            host[i] = o;
        }
    });
}

int odegpu_batch_write_outcomes(odegpu_batch* b, const odegpu_outcome* host) {
    return guarded([&] {
        check_batch(b);
        if (!host) throw_invalid("null argument");
        DeviceGuard g(b->device);
        const size_t n = size_t(b->dims.batch_capacity);
        std::vector<double> ft(n), ss(n);
        std::vector<Index> acc(n), rej(n), det(n), sf(n);
        std::vector<std::uint8_t> rs(n);
        for (size_t i = 0; i < n; ++i) {
            ft[i] = host[i].final_t;
            rs[i] = host[i].reason;
            acc[i] = host[i].accepted_steps;
            rej[i] = host[i].rejected_steps;
            det[i] = host[i].event_detections;
            sf[i] = host[i].secant_failures;
            ss[i] = host[i].smallest_step;
        }
        CK(cudaMemcpyAsync(b->a.final_t, ft.data(), n * 8, cudaMemcpyHostToDevice, b->stream));
        CK(cudaMemcpyAsync(b->a.reason, rs.data(), n, cudaMemcpyHostToDevice, b->stream));
        CK(cudaMemcpyAsync(b->a.accepted, acc.data(), n * 8, cudaMemcpyHostToDevice, b->stream));
        CK(cudaMemcpyAsync(b->a.rejected, rej.data(), n * 8, cudaMemcpyHostToDevice, b->stream));
        CK(cudaMemcpyAsync(b->a.detections, det.data(), n * 8, cudaMemcpyHostToDevice, b->stream));
        CK(cudaMemcpyAsync(b->a.secant_failures, sf.data(), n * 8, cudaMemcpyHostToDevice, b->stream));
        CK(cudaMemcpyAsync(b->a.smallest_step, ss.data(), n * 8, cudaMemcpyHostToDevice, b->stream));
        CK(cudaStreamSynchronize(b->stream));
    });
}

int odegpu_batch_reset_outcomes(odegpu_batch* b) {
    return guarded([&] {
        check_batch(b);
        DeviceGuard g(b->device);
        reset_outcomes_kernel<<<grid_for(b, b->dims.batch_capacity, 256), 256, 0, b->stream>>>(
            b->a, 0, b->dims.batch_capacity);
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(b->stream));
    });
}

int odegpu_solve(odegpu_batch* b, const odegpu_model* m, const odegpu_solver_config* cfg,
                 const odegpu_ode_controls* ode, const odegpu_event_controls* ev) {
    return guarded([&] {
        const dev::Controls c = prepare_solve(b, m, cfg, ode, ev);
        DeviceGuard g(b->device);
        enqueue_time_check(b);
        launch_model(b, *m, cfg->algorithm, c);
        raise_if_bad(b); // synchronous, like solve.hpp:143
    });
}

int odegpu_solve_iteratively(odegpu_batch* b, const odegpu_model* m, const odegpu_solver_config* cfg,
                             const odegpu_ode_controls* ode, const odegpu_event_controls* ev,
                             odegpu_index iterations, odegpu_sink sink, void* user) {
    int sink_rc = 0;
    const int rc = guarded([&] {
        if (iterations < 1) throw_invalid("solve_iteratively: iterations must be >= 1"); // solve.hpp:137
        const dev::Controls c = prepare_solve(b, m, cfg, ode, ev);
        DeviceGuard g(b->device);
        for (Index it = 0; it < iterations; ++it) {
            enqueue_time_check(b);
            launch_model(b, *m, cfg->algorithm, c);
            if (sink) {
                raise_if_bad(b);
                sink_rc = sink(it, b, user);
                if (sink_rc != 0) return;
            }
        }
        if (!sink) raise_if_bad(b); // a skipped iteration leaves every later one skipped
    });
    return rc != 0 ? rc : sink_rc;
}

int odegpu_batch_sync(odegpu_batch* b) {
    return guarded([&] {
        check_batch(b);
        DeviceGuard g(b->device);
        CK(cudaStreamSynchronize(b->stream));
    });
}

int64_t odegpu_batch_launch_count(const odegpu_batch* b) { return b ? b->launches : 0; }

int odegpu_batch_diagnostics(odegpu_batch* b, odegpu_diagnostics* out) {
    return guarded([&] {
        check_batch(b);
        if (!out) throw_invalid("null argument");
        DeviceGuard g(b->device);
        CK(cudaMemsetAsync(b->diag, 0, 9 * sizeof(unsigned long long), b->stream));
        diagnostics_kernel<<<grid_for(b, b->dims.batch_capacity, 256), 256, 0, b->stream>>>(b->a, b->diag);
        CK(cudaGetLastError());
        ++b->launches;
        unsigned long long h[9];
        CK(cudaMemcpyAsync(h, b->diag, sizeof h, cudaMemcpyDeviceToHost, b->stream));
        CK(cudaStreamSynchronize(b->stream));
        out->accepted_steps = static_cast<Index>(h[0]);
        out->rejected_steps = static_cast<Index>(h[1]);
        out->event_detections = static_cast<Index>(h[2]);
        out->secant_failures = static_cast<Index>(h[3]);
        for (int k = 0; k < 4; ++k) out->reason_counts[k] = static_cast<Index>(h[4 + k]);
        out->max_trial_steps = static_cast<Index>(h[8]);
    });
}

int odegpu_batch_last_kernel_ms(odegpu_batch* b, double* ms) {
    return guarded([&] {
        check_batch(b);
        if (!ms) throw_invalid("null argument");
        if (!b->timed) throw_invalid("no solve kernel has run on this batch");
        DeviceGuard g(b->device);
        CK(cudaEventSynchronize(b->ev_stop));
        float f = 0;
        CK(cudaEventElapsedTime(&f, b->ev_start, b->ev_stop));
        *ms = f;
    });
}

int odegpu_dfma_peak(int device, int blocks, int threads, int iters, double* lane_dfma_per_s, double* seconds) {
    return guarded([&] {
        if (blocks < 1 || threads < 1 || iters < 1) throw_invalid("dfma_peak: bad geometry");
        DeviceGuard g(device);
        double* out = nullptr;
        cudaEvent_t e0, e1;
        CK(cudaMalloc(&out, 8));
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        dfma_peak_kernel<<<blocks, threads>>>(out, iters, 1.0); // warm-up
        CK(cudaGetLastError());
        CK(cudaEventRecord(e0));
        dfma_peak_kernel<<<blocks, threads>>>(out, iters, 1.0);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        cudaFree(out);
        const double lanes = double(blocks) * threads * double(iters) * 32.0;
        if (seconds) *seconds = ms * 1e-3;
        if (lane_dfma_per_s) *lane_dfma_per_s = lanes / (ms * 1e-3);
    });
}

} // extern "C"
