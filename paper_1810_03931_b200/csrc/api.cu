// api.cu — the C ABI (include/odegpu.h): device-resident SoA batches,
// pool<->batch copies, validation with the reference's messages, solve
// dispatch. Kernels live in kernels.cu and the models_*.cu units; the
// chunked pool pipeline in pipeline.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <unordered_set>
#include <vector>

#include <cstdlib>

#include "internal.cuh"

using namespace odegpu;
using namespace odegpu::detail;

static_assert(sizeof(odegpu_outcome) == 56, "odegpu_outcome must match odensemble::SystemOutcome");

namespace odegpu::detail {

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

odegpu_system_dims dims_of(const odegpu_model& m) {
    odegpu_system_dims d{};
    if (family_dims_duffing(m, &d) || family_dims_keller_miksis(m, &d) || family_dims_valve(m, &d) ||
        family_dims_fakes(m, &d))
        return d;
    throw_unsupported("unknown model id " + std::to_string(m.id));
}

bool keeps_time_domain(const odegpu_model& m) {
    odegpu_system_dims d{};
    bool keeps = false;
    if (family_dims_duffing(m, &d, &keeps) || family_dims_keller_miksis(m, &d, &keeps) ||
        family_dims_valve(m, &d, &keeps) || family_dims_fakes(m, &d, &keeps))
        return keeps;
    throw_unsupported("unknown model id " + std::to_string(m.id));
}

bool fusable_iterations(const odegpu_model& m) {
    odegpu_system_dims d{};
    bool keeps = false, fusable = false;
    if (family_dims_duffing(m, &d, &keeps, &fusable) || family_dims_keller_miksis(m, &d, &keeps, &fusable) ||
        family_dims_valve(m, &d, &keeps, &fusable) || family_dims_fakes(m, &d, &keeps, &fusable))
        return fusable;
    throw_unsupported("unknown model id " + std::to_string(m.id));
}

void launch_model(odegpu_batch* b, const odegpu_model& m, int algorithm, const dev::Controls& c) {
    if (family_launch_duffing(b, m, algorithm, c) || family_launch_keller_miksis(b, m, algorithm, c) ||
        family_launch_valve(b, m, algorithm, c) || family_launch_fakes(b, m, algorithm, c))
        return;
    throw_unsupported("unknown model id " + std::to_string(m.id));
}

// solve.hpp:145-157: validation that needs no device data, plus control
// materialisation into the kernel-parameter struct.
dev::Controls prepare_solve(const odegpu_batch_dims& d, const odegpu_model* m, const odegpu_solver_config* cfg,
                            const odegpu_ode_controls* ode, const odegpu_event_controls* ev) {
    if (!m) throw_invalid("solve: null argument");
    return validate_solve(d, dims_of(*m), cfg, ode, ev);
}

dev::Controls validate_solve(const odegpu_batch_dims& d, const odegpu_system_dims& sys,
                             const odegpu_solver_config* cfg, const odegpu_ode_controls* ode,
                             const odegpu_event_controls* ev) {
    if (!cfg || !ode) throw_invalid("solve: null argument");
    if (sys.system_dim != d.system_dim || sys.param_count != d.param_count || sys.event_count != d.event_count ||
        sys.accessory_count != d.accessory_count)
        throw_invalid("solve: definition and batch dimensions disagree");
    if (cfg->initial_time_step <= 0) throw_invalid("solve: initial_time_step must be > 0");
    if (cfg->tile_size < 1) throw_invalid("solve: tile_size must be >= 1");
    if (cfg->algorithm != ODEGPU_RK4 && cfg->algorithm != ODEGPU_RKCK45) throw_invalid("solve: unknown algorithm");
    if (cfg->algorithm != ODEGPU_RK4 && cfg->initial_time_step > ode->max_step)
        throw_invalid("solve: initial_time_step exceeds max_step");
    if (sys.system_dim > dev::kMaxDim || sys.event_count > dev::kMaxEvents)
        throw_unsupported("solve: model wider than the device controls");
    if (!ode->rel_tol || !ode->abs_tol) throw_invalid("solve: null tolerance arrays");
    if (sys.event_count > 0 && (!ev || !ev->direction || !ev->tolerance || !ev->stop_condition))
        throw_invalid("solve: event controls missing");

    return dev::controls_from(sys, *cfg, *ode, ev);
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
    // `components` rows of `count` doubles (batch.cpp:55-63 as one 2D copy)
    CK(cudaMemcpy2DAsync(dst + dst_start, size_t(dst_stride) * sizeof(Real), src + src_start,
                         size_t(src_stride) * sizeof(double), size_t(count) * sizeof(Real), size_t(components),
                         cudaMemcpyHostToDevice, s));
}

void copy_d2h_strided(double* dst, Index dst_stride, Index dst_start, const Real* src, Index src_stride,
                      Index src_start, Index count, Index components, cudaStream_t s) {
    if (count == 0 || components == 0) return;
    CK(cudaMemcpy2DAsync(dst + dst_start, size_t(dst_stride) * sizeof(double), src + src_start,
                         size_t(src_stride) * sizeof(Real), size_t(count) * sizeof(Real), size_t(components),
                         cudaMemcpyDeviceToHost, s));
}

namespace {
size_t align_up(size_t v) { return (v + 255) & ~size_t(255); }
} // namespace

odegpu_batch* batch_create(const odegpu_batch_dims& dims, int device) {
    // BatchDims::validate (pool.hpp:67-73)
    if (dims.batch_capacity < 1) throw_invalid("BatchDims: batch_capacity must be >= 1");
    if (dims.batch_capacity > Index(0xffffffff)) // lanes address slots in 32 bits (solver.cuh ColdState)
        throw_invalid("BatchDims: batch_capacity must be < 2^32 on the device");
    if (dims.system_dim < 1) throw_invalid("BatchDims: system_dim must be >= 1");
    if (dims.param_count < 0) throw_invalid("BatchDims: param_count must be >= 0");
    if (dims.event_count < 0) throw_invalid("BatchDims: event_count must be >= 0");
    if (dims.accessory_count < 0) throw_invalid("BatchDims: accessory_count must be >= 0");
    DeviceGuard g(device);
    auto* b = new odegpu_batch;
    b->dims = dims;
    b->device = device;
    // tuning / experiment override of the default fetch order (0 natural,
    // 1 cost, 2 auto) for batches the caller does not see (pipeline slots)
    if (const char* env = std::getenv("ODEGPU_FETCH_ORDER"); env && env[0] >= '0' && env[0] <= '2' && !env[1])
        b->order_mode = env[0] - '0';
    try {
        CK(cudaDeviceGetAttribute(&b->num_sms, cudaDevAttrMultiProcessorCount, device));
        CK(cudaStreamCreateWithFlags(&b->own_stream, cudaStreamNonBlocking));
        b->stream = b->own_stream;
        const size_t n = size_t(dims.batch_capacity);
        const size_t sizes[] = {2 * n * 8,
                                size_t(dims.system_dim) * n * 8,
                                size_t(dims.param_count) * n * 8,
                                size_t(dims.accessory_count) * n * 8,
                                n * 8,                      // final_t
                                n,                          // reason
                                n * 8, n * 8, n * 8, n * 8, // counters
                                n * 8,                      // smallest_step
                                8, 16, 128, 8};             // work, first_bad + trig flag, diag, trial steps
        constexpr int kArrays = sizeof(sizes) / sizeof(sizes[0]);
        size_t total = 0;
        for (size_t s : sizes) total += align_up(s);
        CK(cudaMalloc(&b->block, total));
        CK(cudaMemsetAsync(b->block, 0, total, b->stream));
        char* p = static_cast<char*>(b->block);
        void* ptrs[kArrays];
        for (int i = 0; i < kArrays; ++i) {
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
        b->trial_steps = static_cast<unsigned long long*>(ptrs[14]);
        b->a.n = dims.batch_capacity;
        b->a.count = dims.batch_capacity;
        CK(cudaEventCreate(&b->ev_start));
        CK(cudaEventCreate(&b->ev_stop));
        CK(cudaMallocHost(&b->host_flag, sizeof(unsigned long long)));
        launch_reset_outcomes(b, 0, dims.batch_capacity);
        CK(cudaStreamSynchronize(b->stream));
    } catch (...) {
        odegpu_batch_destroy(b);
        throw;
    }
    return b;
}

} // namespace odegpu::detail

// ============================================================ C ABI

extern "C" {

int odegpu_abi_version(void) { return ODEGPU_ABI_VERSION; }

int odegpu_build_flags(void) {
#if defined(ODEGPU_PARITY_BUILD) && ODEGPU_PARITY_BUILD
    return ODEGPU_BUILD_PARITY;
#else
    return 0;
#endif
}

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
        *out = batch_create(*dims, device);
    });
}

void odegpu_batch_destroy(odegpu_batch* b) {
    if (!b) return;
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(b->device);
    if (b->stream) cudaStreamSynchronize(b->stream);
    if (b->block) cudaFree(b->block);
    if (b->order_block) cudaFree(b->order_block);
    if (b->log_block) cudaFree(b->log_block);
    if (b->host_flag) cudaFreeHost(b->host_flag);
    if (b->ev_start) cudaEventDestroy(b->ev_start);
    if (b->ev_stop) cudaEventDestroy(b->ev_stop);
    if (b->own_stream) cudaStreamDestroy(b->own_stream);
    release_batch_stage(b);
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

int odegpu_batch_set_fetch_order(odegpu_batch* b, int32_t mode) {
    return guarded([&] {
        check_batch(b);
        if (mode < ODEGPU_FETCH_NATURAL || mode > ODEGPU_FETCH_AUTO) throw_invalid("unknown fetch order mode");
        b->order_mode = mode;
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
        launch_reset_outcomes(b, spec->start_in_batch, n); // batch.cpp:102-103
        CK(cudaStreamSynchronize(b->stream));             // the pool may be reused on return
    });
}

int odegpu_random_set(odegpu_batch* b, const odegpu_pool_view* pool, const odegpu_index* ib,
                      const odegpu_index* ip, odegpu_index count, int32_t copy_mode) {
    return guarded([&] {
        check_batch(b);
        if (!pool) throw_invalid("null argument");
        check_dims_agree(b->dims, pool->dims); // batch.cpp:107-117
        if (count < 0 || (count > 0 && (!ib || !ip))) throw_invalid("random_set: index lists differ in length");
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
        for (int32_t prop = 0; prop <= ODEGPU_PROP_ACCESSORIES; ++prop) // before any allocation
            if (wants(copy_mode, prop) && components_of(b->dims, prop) > 0 && !pool_ptr(pool, prop))
                throw_invalid("random_set: pool array missing");
        DeviceGuard g(b->device);
        const Index np = pool->dims.problem_size;
        // gather on the host into one staging block, one H2D, scatter on device
        Index total_comps = 0;
        for (int32_t prop = 0; prop <= ODEGPU_PROP_ACCESSORIES; ++prop)
            if (wants(copy_mode, prop)) total_comps += components_of(b->dims, prop);
        std::vector<double> staged(size_t(total_comps * count) + 1);
        Index* d_idx = nullptr;
        double* d_staged = nullptr;
        // freed on every path, a CUDA error after the allocations included
        struct Scratch {
            Index** idx;
            double** staged;
            cudaStream_t s;
            ~Scratch() {
                if (*idx) cudaFreeAsync(*idx, s);
                if (*staged) cudaFreeAsync(*staged, s);
            }
        } scratch{&d_idx, &d_staged, b->stream};
        CK(cudaMallocAsync(reinterpret_cast<void**>(&d_idx), size_t(count) * sizeof(Index), b->stream));
        CK(cudaMallocAsync(reinterpret_cast<void**>(&d_staged), staged.size() * sizeof(double), b->stream));
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
            launch_scatter_rows(b, property_ptr(b, prop), d_idx, d_staged + off, count, comps);
            off += comps * count;
        }
        launch_reset_rows(b, d_idx, count); // batch.cpp:134
        CK(cudaFreeAsync(d_idx, b->stream));
        d_idx = nullptr;
        CK(cudaFreeAsync(d_staged, b->stream));
        d_staged = nullptr;
        CK(cudaStreamSynchronize(b->stream)); // `staged` is pageable host memory
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
        copy_d2h_strided(host, host_stride, 0, property_ptr(b, property), b->dims.batch_capacity, start, count,
                         comps, b->stream);
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
        download_outcomes(b, 0, b->dims.batch_capacity, host);
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
        launch_reset_outcomes(b, 0, b->dims.batch_capacity);
        CK(cudaStreamSynchronize(b->stream));
    });
}

int odegpu_batch_copy(odegpu_batch* dst, const odegpu_batch* src) {
    return guarded([&] {
        check_batch(dst);
        check_batch(src);
        const auto &a = dst->dims, &c = src->dims;
        if (a.batch_capacity != c.batch_capacity || a.system_dim != c.system_dim || a.param_count != c.param_count ||
            a.event_count != c.event_count || a.accessory_count != c.accessory_count)
            throw_invalid("batch_copy: batches differ in dimensions");
        DeviceGuard g(dst->device);
        CK(cudaStreamSynchronize(src->stream));
        // the data arrays and outcome fields occupy the same offsets in both blocks
        const size_t bytes = static_cast<const char*>(static_cast<const void*>(src->a.work)) -
                             static_cast<const char*>(src->block);
        CK(cudaMemcpyAsync(dst->block, src->block, bytes, cudaMemcpyDeviceToDevice, dst->stream));
        CK(cudaStreamSynchronize(dst->stream));
    });
}

int odegpu_solve(odegpu_batch* b, const odegpu_model* m, const odegpu_solver_config* cfg,
                 const odegpu_ode_controls* ode, const odegpu_event_controls* ev) {
    return guarded([&] {
        check_batch(b);
        const dev::Controls c = prepare_solve(b->dims, m, cfg, ode, ev);
        DeviceGuard g(b->device);
        b->a.count = b->dims.batch_capacity;
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
        check_batch(b);
        if (iterations < 1) throw_invalid("solve_iteratively: iterations must be >= 1"); // solve.hpp:137
        const dev::Controls c = prepare_solve(b->dims, m, cfg, ode, ev);
        DeviceGuard g(b->device);
        b->a.count = b->dims.batch_capacity;
        if (!sink) {
            // no host round trip between iterations: models whose finalize
            // keeps the time domain valid run them fused, every system solved
            // `iterations` times in a row by one lane in as few launches as
            // possible (hooks.hpp kFusableIterations); the t1 < t0 check of
            // each launch covers the iterations it fuses
            for (Index it = 0; it < iterations;) {
                enqueue_time_check(b);
                b->fuse_request = iterations - it;
                launch_model(b, *m, cfg->algorithm, c);
                it += b->fused_done;
            }
            raise_if_bad(b); // a skipped iteration leaves every later one skipped
            return;
        }
        for (Index it = 0; it < iterations; ++it) {
            enqueue_time_check(b);
            launch_model(b, *m, cfg->algorithm, c);
            raise_if_bad(b);
            sink_rc = sink(it, b, user);
            if (sink_rc != 0) return;
        }
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

int odegpu_batch_set_detection_log(odegpu_batch* b, odegpu_index capacity) {
    return guarded([&] {
        check_batch(b);
        if (capacity < 0) throw_invalid("detection log: capacity must be >= 0");
        DeviceGuard g(b->device);
        CK(cudaStreamSynchronize(b->stream));
        if (b->log_block) CK(cudaFree(b->log_block));
        b->log_block = nullptr;
        auto& a = b->a;
        a.log_count = nullptr;
        a.log_capacity = 0;
        if (capacity == 0) return;
        const size_t c = size_t(capacity), dim = size_t(b->dims.system_dim);
        const size_t sizes[] = {8, c * 4, c * 4, c * 4, c * 4, c * 8, c * 8, c * 8, c * 8, dim * c * 8, dim * c * 8};
        size_t total = 0;
        for (size_t v : sizes) total += align_up(v);
        CK(cudaMalloc(&b->log_block, total));
        char* q = static_cast<char*>(b->log_block);
        void* ptr[11];
        for (int i = 0; i < 11; ++i) {
            ptr[i] = q;
            q += align_up(sizes[i]);
        }
        a.log_count = static_cast<unsigned long long*>(ptr[0]);
        a.log_system = static_cast<unsigned*>(ptr[1]);
        a.log_event = static_cast<int*>(ptr[2]);
        a.log_kind = static_cast<int*>(ptr[3]);
        a.log_in_zone = static_cast<int*>(ptr[4]);
        a.log_counter = static_cast<long long*>(ptr[5]);
        a.log_sequence = static_cast<long long*>(ptr[6]);
        a.log_t = static_cast<Real*>(ptr[7]);
        a.log_value = static_cast<Real*>(ptr[8]);
        a.log_y_pre = static_cast<Real*>(ptr[9]);
        a.log_y_post = static_cast<Real*>(ptr[10]);
        a.log_capacity = capacity;
        CK(cudaMemsetAsync(a.log_count, 0, 8, b->stream));
    });
}

int odegpu_batch_read_detection_log(odegpu_batch* b, odegpu_detection* records, double* y_pre, double* y_post,
                                    odegpu_index capacity, odegpu_index* count, odegpu_index* total) {
    return guarded([&] {
        check_batch(b);
        if (!count || !total) throw_invalid("null argument");
        const auto& a = b->a;
        if (!a.log_count) throw_invalid("detection log: not enabled (odegpu_batch_set_detection_log)");
        DeviceGuard g(b->device);
        unsigned long long n_all = 0;
        CK(cudaMemcpyAsync(&n_all, a.log_count, 8, cudaMemcpyDeviceToHost, b->stream));
        CK(cudaStreamSynchronize(b->stream));
        const Index stored = std::min<Index>(static_cast<Index>(n_all), a.log_capacity);
        *total = static_cast<Index>(n_all);
        const Index n = std::min<Index>(stored, std::max<Index>(capacity, 0));
        *count = 0;
        if (n == 0) return;
        if (!records) throw_invalid("null argument");
        const size_t c = size_t(stored), dim = size_t(b->dims.system_dim);
        std::vector<unsigned> sys(c);
        std::vector<int> ev(c), kind(c), zone(c);
        std::vector<long long> cnt(c), seq(c);
        std::vector<Real> t(c), v(c), pre(dim * c), post(dim * c);
        auto get = [&](void* dst, const void* src, size_t bytes) {
            CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, b->stream));
        };
        get(sys.data(), a.log_system, c * 4);
        get(ev.data(), a.log_event, c * 4);
        get(kind.data(), a.log_kind, c * 4);
        get(zone.data(), a.log_in_zone, c * 4);
        get(cnt.data(), a.log_counter, c * 8);
        get(seq.data(), a.log_sequence, c * 8);
        get(t.data(), a.log_t, c * 8);
        get(v.data(), a.log_value, c * 8);
        for (size_t j = 0; j < dim; ++j) {
            get(pre.data() + j * c, a.log_y_pre + j * size_t(a.log_capacity), c * 8);
            get(post.data() + j * c, a.log_y_post + j * size_t(a.log_capacity), c * 8);
        }
        CK(cudaStreamSynchronize(b->stream));
        // slots are claimed in completion order across lanes: hand records
        // out per system in the order its driver made them
        std::vector<size_t> idx(c);
        for (size_t i = 0; i < c; ++i) idx[i] = i;
        std::sort(idx.begin(), idx.end(), [&](size_t x, size_t y) {
            return sys[x] != sys[y] ? sys[x] < sys[y] : seq[x] < seq[y];
        });
        for (Index k = 0; k < n; ++k) {
            const size_t i = idx[size_t(k)];
            odegpu_detection& d = records[k];
            d.system = sys[i];
            d.event_index = ev[i];
            d.counter = cnt[i];
            d.sequence = seq[i];
            d.t = t[i];
            d.value = v[i];
            d.kind = kind[i];
            d.in_zone = zone[i];
            for (size_t j = 0; j < dim; ++j) {
                if (y_pre) y_pre[size_t(k) * dim + j] = pre[j * c + i];
                if (y_post) y_post[size_t(k) * dim + j] = post[j * c + i];
            }
        }
        *count = n;
    });
}

int64_t odegpu_batch_launch_count(const odegpu_batch* b) { return b ? b->launches : 0; }

int odegpu_batch_device(const odegpu_batch* b) { return b ? b->device : -1; }

int odegpu_model_keeps_time_domain(const odegpu_model* m, int* keeps) {
    return guarded([&] {
        if (!m || !keeps) throw_invalid("null argument");
        *keeps = keeps_time_domain(*m) ? 1 : 0;
    });
}

int odegpu_batch_diagnostics(odegpu_batch* b, odegpu_diagnostics* out) {
    return guarded([&] {
        check_batch(b);
        if (!out) throw_invalid("null argument");
        DeviceGuard g(b->device);
        launch_diagnostics(b);
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

int odegpu_batch_trial_steps(odegpu_batch* b, odegpu_index* total, int reset) {
    return guarded([&] {
        check_batch(b);
        if (!total) throw_invalid("null argument");
        DeviceGuard g(b->device);
        unsigned long long h = 0;
        CK(cudaMemcpyAsync(&h, b->trial_steps, sizeof h, cudaMemcpyDeviceToHost, b->stream));
        if (reset) CK(cudaMemsetAsync(b->trial_steps, 0, sizeof h, b->stream));
        CK(cudaStreamSynchronize(b->stream));
        *total = static_cast<Index>(h);
    });
}

int odegpu_batch_trig_certified(odegpu_batch* b, int* certified) {
    return guarded([&] {
        check_batch(b);
        if (!certified) throw_invalid("null argument");
        DeviceGuard g(b->device);
        unsigned long long f[2] = {0, 0};
        CK(cudaMemcpyAsync(f, b->first_bad, sizeof(f), cudaMemcpyDeviceToHost, b->stream));
        CK(cudaStreamSynchronize(b->stream));
        *certified = (b->timed && f[1] == 0) ? 1 : 0;
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
        const double r = run_dfma_peak(blocks, threads, iters, seconds);
        if (lane_dfma_per_s) *lane_dfma_per_s = r;
    });
}

} // extern "C"

extern "C" int odegpu_custom_begin(odegpu_batch* b, const odegpu_system_dims* dims, const odegpu_solver_config* cfg,
                                   const odegpu_ode_controls* ode, const odegpu_event_controls* ev,
                                   odegpu_device_view* view) {
    return guarded([&] {
        check_batch(b);
        if (!dims || !view) throw_invalid("solve: null argument");
        validate_solve(b->dims, *dims, cfg, ode, ev); // solve.hpp:145-157, same messages
        DeviceGuard g(b->device);
        b->a.count = b->dims.batch_capacity;
        enqueue_time_check(b);
        CK(cudaMemsetAsync(b->a.work, 0, sizeof(unsigned long long), b->stream));
        const auto& a = b->a;
        *view = odegpu_device_view{a.td,          a.state,      a.params,          a.acc,
                                   a.final_t,     a.reason,     a.accepted,        a.rejected,
                                   a.detections,  a.secant_failures, a.smallest_step, a.n,
                                   a.count,       a.work,       b->first_bad,      b->stream,
                                   b->device,     b->num_sms};
        ++b->launches; // the caller's solve kernel
    });
}

extern "C" int odegpu_custom_end(odegpu_batch* b) {
    return guarded([&] {
        check_batch(b);
        DeviceGuard g(b->device);
        CK(cudaGetLastError()); // the caller's launch
        raise_if_bad(b);
    });
}

extern "C" int odegpu_math_check(int fn, odegpu_index n, const double* x, const double* y, double* mine,
                                 double* ref) {
    return guarded([&] {
        if (fn < 0 || fn > 12 || n < 0 || !x || !mine || !ref || ((fn == 1 || fn == 6 || fn == 7 || fn == 12) && !y))
            throw_invalid("math_check: bad arguments");
        if (n > 0) run_math_check(fn, n, x, y, mine, ref);
    });
}
