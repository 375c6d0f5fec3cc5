// device_pool.cu — a problem pool kept in HBM.
//
// The reference's ProblemPool (pool.hpp:12-64) is host storage that
// linear_set / random_set (batch.cpp:78-135) copy into a SolverBatch. Here
// the pool itself can live on the device: 180 GB of HBM hold ~50x the
// largest BASELINE pool (2^24 Keller-Miksis systems, 3.3 GB), so pools of
// up to ~10^9 small systems never cross PCIe. On top of it:
//  * linear_set / random_set from the device pool — device gathers with the
//    reference's validation and messages, outcomes of the copied slots reset
//    (batch.cpp:102-103, 134);
//  * store — the reverse copy, batch slots back into pool rows (what a scan
//    driver does with the end points of a chunk);
//  * odegpu_device_pool_solve — the chunked solve of the whole pool through
//    device batches with COST-CLUSTERED RE-BATCHING (PAPER.md:833:
//    "organize the problem so that the threads in a warp have similar
//    parameter values ... similar collapse strength"). After a solve the
//    pool keeps every system's RK steps; the next clustered solve sorts the
//    pool longest first and deals it round-robin into the chunks, so every
//    chunk gets the same cost profile (no chunk of only long systems, no
//    chunk of only short ones) and takes its systems longest first — a warp's
//    lanes meet systems of similar cost together and the long ones never form
//    a chunk's tail (list scheduling, longest processing time first). Results
//    never depend on the chunking (each system's arithmetic is its own):
//    tests/test_gpu_device_pool.py checks them bit for bit against one
//    resident batch.
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <unordered_set>
#include <vector>

#include "internal.cuh"

/// The pool object: SoA arrays of stride N (pool.hpp:12-23), the outcome
/// record of each system's last pool solve, its cost, and the working set of
/// pool solves (two device batches, the permutation).
struct odegpu_device_pool {
    odegpu_pool_dims dims{};
    int device = 0;
    cudaStream_t stream = nullptr;
    void* block = nullptr;
    odegpu::Real *td = nullptr, *state = nullptr, *params = nullptr, *acc = nullptr;
    odegpu::Real *final_t = nullptr, *smallest = nullptr;
    std::uint8_t* reason = nullptr;
    odegpu::Index *accepted = nullptr, *rejected = nullptr, *detections = nullptr, *secant_failures = nullptr;
    unsigned* cost = nullptr; // RK evaluations of the last pool solve (0: not solved yet)
    bool has_cost = false;
    // pool-solve working set (lazy)
    odegpu_batch* batch[2] = {nullptr, nullptr};
    odegpu_model batch_model{};
    odegpu::Index batch_cap = 0;
    void* order_block = nullptr; // permutation + sort keys + CUB scratch
    std::size_t order_bytes = 0;

    ~odegpu_device_pool() {
        if (stream) cudaStreamSynchronize(stream);
        for (odegpu_batch* b : batch)
            if (b) odegpu_batch_destroy(b);
        if (order_block) cudaFree(order_block);
        if (block) cudaFree(block);
        if (stream) cudaStreamDestroy(stream);
    }
};

namespace odegpu::detail {
namespace {

std::size_t align_up(std::size_t v) { return (v + 255) & ~std::size_t(255); }

Real* pool_array(odegpu_device_pool* p, int32_t prop) {
    switch (prop) {
    case ODEGPU_PROP_TIME_DOMAIN: return p->td;
    case ODEGPU_PROP_STATE: return p->state;
    case ODEGPU_PROP_PARAMETERS: return p->params;
    case ODEGPU_PROP_ACCESSORIES: return p->acc;
    default: return nullptr;
    }
}

Index pool_components(const odegpu_pool_dims& d, int32_t prop) {
    switch (prop) {
    case ODEGPU_PROP_TIME_DOMAIN: return 2;
    case ODEGPU_PROP_STATE: return d.system_dim;
    case ODEGPU_PROP_PARAMETERS: return d.param_count;
    case ODEGPU_PROP_ACCESSORIES: return d.accessory_count;
    default: return 0;
    }
}

/// dst[row_d(j) + c*nd] = src[row_s(j) + c*ns] for j < count, c < comps;
/// a null index list means the contiguous rows start + j. Consecutive
/// threads take consecutive j of one component: a contiguous side is read
/// or written coalesced, a permuted side is a gather / scatter of 8-byte
/// rows (HBM-bound either way).
template <class DI, class SI>
__global__ void copy_rows_kernel(Real* dst, Index nd, const DI* dst_idx, Index dst_start, const Real* src, Index ns,
                                 const SI* src_idx, Index src_start, Index count, Index comps) {
    const Index total = count * comps;
    for (Index k = blockIdx.x * static_cast<Index>(blockDim.x) + threadIdx.x; k < total;
         k += static_cast<Index>(gridDim.x) * blockDim.x) {
        const Index c = k / count, j = k - c * count;
        const Index rd = dst_idx ? static_cast<Index>(dst_idx[j]) : dst_start + j;
        const Index rs = src_idx ? static_cast<Index>(src_idx[j]) : src_start + j;
        dst[rd + c * nd] = src[rs + c * ns];
    }
}

template <class DI, class SI>
void copy_rows(Real* dst, Index nd, const DI* dst_idx, Index dst_start, const Real* src, Index ns, const SI* src_idx,
               Index src_start, Index count, Index comps, int num_sms, cudaStream_t s) {
    if (count <= 0 || comps <= 0) return;
    const Index work = count * comps;
    const int grid = static_cast<int>(std::max<Index>(1, std::min<Index>((work + 255) / 256, Index(num_sms) * 16)));
    copy_rows_kernel<DI, SI><<<grid, 256, 0, s>>>(dst, nd, dst_idx, dst_start, src, ns, src_idx, src_start, count,
                                                  comps);
    CK(cudaGetLastError());
}

/// The pool's outcome columns, as a kernel argument.
struct PoolOutcomes {
    Real *final_t, *smallest;
    std::uint8_t* reason;
    Index *accepted, *rejected, *detections, *secant_failures;
    unsigned* cost;
};

/// Outcome records of batch slots [0, count) into pool rows perm[j] (or
/// start + j), and each system's cost (accepted + rejected steps of the
/// solve, saturating at 2^32 - 1).
template <class I>
__global__ void store_outcomes_kernel(dev::BatchArrays b, Index count, const I* rows, Index start, PoolOutcomes p) {
    for (Index j = blockIdx.x * static_cast<Index>(blockDim.x) + threadIdx.x; j < count;
         j += static_cast<Index>(gridDim.x) * blockDim.x) {
        const Index r = rows ? static_cast<Index>(rows[j]) : start + j;
        p.final_t[r] = b.final_t[j];
        p.reason[r] = b.reason[j];
        p.accepted[r] = b.accepted[j];
        p.rejected[r] = b.rejected[j];
        p.detections[r] = b.detections[j];
        p.secant_failures[r] = b.secant_failures[j];
        p.smallest[r] = b.smallest_step[j];
        const unsigned long long c =
            static_cast<unsigned long long>(b.accepted[j]) + static_cast<unsigned long long>(b.rejected[j]);
        p.cost[r] = c > 0xffffffffull ? 0xffffffffu : static_cast<unsigned>(c);
    }
}

// solve.hpp:159-161 over the whole pool: lowest index with t1 < t0.
__global__ void pool_time_check_kernel(const Real* td, Index n, unsigned long long* first_bad) {
    for (Index i = blockIdx.x * static_cast<Index>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<Index>(gridDim.x) * blockDim.x)
        if (td[i + n] < td[i]) atomicMin(first_bad, static_cast<unsigned long long>(i));
}

// Deals the longest-first permutation round-robin into k chunks: chunk j
// (rows [off_j, off_j + n_j) of `dealt`) holds sorted[j], sorted[j + k], ...
// — every chunk the same cost profile, each in descending cost.
__global__ void deal_kernel(const unsigned* sorted, Index n, Index k, unsigned* dealt) {
    for (Index s = blockIdx.x * static_cast<Index>(blockDim.x) + threadIdx.x; s < n;
         s += static_cast<Index>(gridDim.x) * blockDim.x) {
        const Index j = s % k, i = s / k;
        // chunks 0..r-1 hold q+1 systems, the rest q (n = q k + r)
        const Index q = n / k, r = n % k;
        const Index off = j * q + (j < r ? j : r);
        dealt[off + i] = sorted[s];
    }
}

__global__ void iota_kernel(unsigned* v, Index n) {
    for (Index i = blockIdx.x * static_cast<Index>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<Index>(gridDim.x) * blockDim.x)
        v[i] = static_cast<unsigned>(i);
}

void validate_random(const odegpu_batch_dims& bd, const odegpu_pool_dims& pd, const odegpu_index* ib,
                     const odegpu_index* ip, odegpu_index count, int32_t copy_mode, const char* what) {
    // batch.cpp:106-121, the reference's messages
    const std::string w(what);
    if (count < 0 || (count > 0 && (!ib || !ip))) throw_invalid(w + ": index lists differ in length");
    std::unordered_set<Index> seen;
    for (Index j = 0; j < count; ++j) {
        const Index i = ib[j];
        if (i < 0 || i >= bd.batch_capacity) throw_range(w + ": batch index out of range");
        if (!seen.insert(i).second) throw_invalid(w + ": duplicate batch index " + std::to_string(i));
    }
    for (Index j = 0; j < count; ++j)
        if (ip[j] < 0 || ip[j] >= pd.problem_size) throw_range(w + ": pool index out of range");
    if (copy_mode < ODEGPU_COPY_TIME_DOMAIN || copy_mode > ODEGPU_COPY_ALL) throw_invalid(w + ": unknown copy mode");
}

/// Device copy of two host index lists (stream-ordered allocation).
struct DeviceIndices {
    Index* d = nullptr;
    cudaStream_t s = nullptr;
    DeviceIndices(const odegpu_index* a, const odegpu_index* b, Index count, cudaStream_t st) : s(st) {
        CK(cudaMallocAsync(reinterpret_cast<void**>(&d), std::size_t(2 * count) * sizeof(Index), s));
        CK(cudaMemcpyAsync(d, a, std::size_t(count) * sizeof(Index), cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(d + count, b, std::size_t(count) * sizeof(Index), cudaMemcpyHostToDevice, s));
    }
    ~DeviceIndices() {
        if (d) cudaFreeAsync(d, s);
    }
};

void check_pool(const odegpu_device_pool* p) {
    if (!p) throw_invalid("null device pool");
}

/// Pool -> batch (linear when idx is null, else rows idx[count..2count) of
/// the pool into slots idx[0..count) of the batch), then reset the outcome
/// records of the copied slots.
void gather(odegpu_batch* b, odegpu_device_pool* p, int32_t mode, const Index* bidx, Index bstart, const Index* pidx,
            Index pstart, Index count) {
    for (int32_t prop = ODEGPU_PROP_TIME_DOMAIN; prop <= ODEGPU_PROP_ACCESSORIES; ++prop) {
        if (!wants(mode, prop)) continue;
        const Index comps = components_of(b->dims, prop);
        copy_rows(property_ptr(b, prop), b->dims.batch_capacity, bidx, bstart, pool_array(p, prop),
                  p->dims.problem_size, pidx, pstart, count, comps, b->num_sms, b->stream);
    }
}

} // namespace
} // namespace odegpu::detail

using namespace odegpu;
using namespace odegpu::detail;

extern "C" {

int odegpu_device_pool_create(const odegpu_pool_dims* dims, int device, odegpu_device_pool** out) {
    return guarded([&] {
        if (!dims || !out) throw_invalid("null argument");
        *out = nullptr;
        // PoolDims::validate (pool.hpp:51-56)
        if (dims->problem_size < 1) throw_invalid("PoolDims: problem_size must be >= 1");
        if (dims->system_dim < 1) throw_invalid("PoolDims: system_dim must be >= 1");
        if (dims->param_count < 0) throw_invalid("PoolDims: param_count must be >= 0");
        if (dims->accessory_count < 0) throw_invalid("PoolDims: accessory_count must be >= 0");
        if (dims->problem_size > Index(0xffffffff)) throw_invalid("PoolDims: problem_size must be < 2^32 on the device");
        DeviceGuard g(device);
        auto* p = new odegpu_device_pool;
        try {
            p->dims = *dims;
            p->device = device;
            CK(cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking));
            const std::size_t n = std::size_t(dims->problem_size);
            const std::size_t sizes[] = {2 * n * 8, std::size_t(dims->system_dim) * n * 8,
                                         std::size_t(dims->param_count) * n * 8,
                                         std::size_t(dims->accessory_count) * n * 8,
                                         n * 8, n * 8, n, n * 8, n * 8, n * 8, n * 8, n * 4};
            std::size_t total = 0;
            for (std::size_t v : sizes) total += align_up(v);
            CK(cudaMalloc(&p->block, total));
            CK(cudaMemsetAsync(p->block, 0, total, p->stream));
            char* q = static_cast<char*>(p->block);
            void* ptr[12];
            for (int i = 0; i < 12; ++i) {
                ptr[i] = q;
                q += align_up(sizes[i]);
            }
            p->td = static_cast<Real*>(ptr[0]);
            p->state = static_cast<Real*>(ptr[1]);
            p->params = static_cast<Real*>(ptr[2]);
            p->acc = static_cast<Real*>(ptr[3]);
            p->final_t = static_cast<Real*>(ptr[4]);
            p->smallest = static_cast<Real*>(ptr[5]);
            p->reason = static_cast<std::uint8_t*>(ptr[6]);
            p->accepted = static_cast<Index*>(ptr[7]);
            p->rejected = static_cast<Index*>(ptr[8]);
            p->detections = static_cast<Index*>(ptr[9]);
            p->secant_failures = static_cast<Index*>(ptr[10]);
            p->cost = static_cast<unsigned*>(ptr[11]);
            CK(cudaStreamSynchronize(p->stream));
        } catch (...) {
            delete p;
            throw;
        }
        *out = p;
    });
}

void odegpu_device_pool_destroy(odegpu_device_pool* p) {
    if (!p) return;
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(p->device);
    delete p;
    if (prev >= 0) cudaSetDevice(prev);
}

int odegpu_device_pool_write(odegpu_device_pool* p, int32_t property, odegpu_index start, odegpu_index count,
                             const double* host, odegpu_index host_stride) {
    return guarded([&] {
        check_pool(p);
        const Index comps = pool_components(p->dims, property);
        if (property < ODEGPU_PROP_TIME_DOMAIN || property > ODEGPU_PROP_ACCESSORIES)
            throw_invalid("device pool: unknown property");
        if (start < 0 || count < 0 || start + count > p->dims.problem_size)
            throw_range("device pool: range out of bounds");
        if (host_stride < count) throw_invalid("device pool: host stride < count");
        if (comps == 0 || count == 0) return;
        if (!host) throw_invalid("null argument");
        DeviceGuard g(p->device);
        copy_h2d_strided(pool_array(p, property), p->dims.problem_size, start, host, host_stride, 0, count, comps,
                         p->stream);
        CK(cudaStreamSynchronize(p->stream)); // the host array may be reused on return
        p->has_cost = false;                  // new systems: the last solve's costs no longer describe them
    });
}

int odegpu_device_pool_read(const odegpu_device_pool* cp, int32_t property, odegpu_index start, odegpu_index count,
                            double* host, odegpu_index host_stride) {
    auto* p = const_cast<odegpu_device_pool*>(cp);
    return guarded([&] {
        check_pool(p);
        const Index comps = pool_components(p->dims, property);
        if (property < ODEGPU_PROP_TIME_DOMAIN || property > ODEGPU_PROP_ACCESSORIES)
            throw_invalid("device pool: unknown property");
        if (start < 0 || count < 0 || start + count > p->dims.problem_size)
            throw_range("device pool: range out of bounds");
        if (host_stride < count) throw_invalid("device pool: host stride < count");
        if (comps == 0 || count == 0) return;
        if (!host) throw_invalid("null argument");
        DeviceGuard g(p->device);
        copy_d2h_strided(host, host_stride, 0, pool_array(p, property), p->dims.problem_size, start, count, comps,
                         p->stream);
        CK(cudaStreamSynchronize(p->stream));
    });
}

int odegpu_device_pool_read_outcomes(const odegpu_device_pool* cp, odegpu_index start, odegpu_index count,
                                     odegpu_outcome* out) {
    auto* p = const_cast<odegpu_device_pool*>(cp);
    return guarded([&] {
        check_pool(p);
        if (start < 0 || count < 0 || start + count > p->dims.problem_size)
            throw_range("device pool: range out of bounds");
        if (count == 0) return;
        if (!out) throw_invalid("null argument");
        DeviceGuard g(p->device);
        const std::size_t n = std::size_t(count);
        std::vector<Real> ft(n), sm(n);
        std::vector<Index> a(n), r(n), d(n), sf(n);
        std::vector<std::uint8_t> rs(n);
        auto get = [&](void* dst, const void* src, std::size_t bytes) {
            CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, p->stream));
        };
        get(ft.data(), p->final_t + start, n * 8);
        get(sm.data(), p->smallest + start, n * 8);
        get(a.data(), p->accepted + start, n * 8);
        get(r.data(), p->rejected + start, n * 8);
        get(d.data(), p->detections + start, n * 8);
        get(sf.data(), p->secant_failures + start, n * 8);
        get(rs.data(), p->reason + start, n);
        CK(cudaStreamSynchronize(p->stream));
        for (std::size_t i = 0; i < n; ++i) {
            odegpu_outcome o{};
            o.final_t = ft[i];
            o.reason = rs[i];
            o.accepted_steps = a[i];
            o.rejected_steps = r[i];
            o.event_detections = d[i];
            o.secant_failures = sf[i];
            o.smallest_step = sm[i];
            out[i] = o;
        }
    });
}

int odegpu_linear_set_device(odegpu_batch* b, odegpu_device_pool* p, const odegpu_linear_copy_spec* spec) {
    return guarded([&] {
        check_batch(b);
        check_pool(p);
        if (!spec) throw_invalid("null argument");
        if (b->device != p->device) throw_invalid("linear_set: batch and device pool live on different devices");
        check_dims_agree(b->dims, p->dims); // batch.cpp:79-85
        if (spec->element_count < 0 || spec->start_in_batch < 0 || spec->start_in_pool < 0)
            throw_range("linear_set: negative index or count");
        if (spec->start_in_batch + spec->element_count > b->dims.batch_capacity)
            throw_range("linear_set: range exceeds batch capacity");
        if (spec->start_in_pool + spec->element_count > p->dims.problem_size)
            throw_range("linear_set: range exceeds pool size");
        if (spec->copy_mode < ODEGPU_COPY_TIME_DOMAIN || spec->copy_mode > ODEGPU_COPY_ALL)
            throw_invalid("linear_set: unknown copy mode");
        DeviceGuard g(b->device);
        CK(cudaStreamSynchronize(p->stream)); // pool writes are ordered before
        gather(b, p, spec->copy_mode, static_cast<const Index*>(nullptr), spec->start_in_batch,
               static_cast<const Index*>(nullptr), spec->start_in_pool, spec->element_count);
        launch_reset_outcomes(b, spec->start_in_batch, spec->element_count); // batch.cpp:102-103
        CK(cudaStreamSynchronize(b->stream));
    });
}

int odegpu_random_set_device(odegpu_batch* b, odegpu_device_pool* p, const odegpu_index* ib, const odegpu_index* ip,
                             odegpu_index count, int32_t copy_mode) {
    return guarded([&] {
        check_batch(b);
        check_pool(p);
        if (b->device != p->device) throw_invalid("random_set: batch and device pool live on different devices");
        check_dims_agree(b->dims, p->dims); // batch.cpp:107-117
        validate_random(b->dims, p->dims, ib, ip, count, copy_mode, "random_set");
        if (count == 0) return;
        DeviceGuard g(b->device);
        CK(cudaStreamSynchronize(p->stream));
        DeviceIndices idx(ib, ip, count, b->stream);
        gather(b, p, copy_mode, idx.d, 0, idx.d + count, 0, count);
        launch_reset_rows(b, idx.d, count); // batch.cpp:134
        CK(cudaStreamSynchronize(b->stream));
    });
}

int odegpu_device_pool_store(odegpu_device_pool* p, odegpu_batch* b, const odegpu_index* ib, const odegpu_index* ip,
                             odegpu_index count, int32_t copy_mode) {
    return guarded([&] {
        check_batch(b);
        check_pool(p);
        if (b->device != p->device) throw_invalid("store: batch and device pool live on different devices");
        check_dims_agree(b->dims, p->dims);
        validate_random(b->dims, p->dims, ib, ip, count, copy_mode, "store");
        {
            std::unordered_set<Index> rows; // scattered rows must be distinct
            for (Index j = 0; j < count; ++j)
                if (!rows.insert(ip[j]).second) throw_invalid("store: duplicate pool index " + std::to_string(ip[j]));
        }
        if (count == 0) return;
        DeviceGuard g(b->device);
        CK(cudaStreamSynchronize(p->stream));
        DeviceIndices idx(ib, ip, count, b->stream);
        for (int32_t prop = ODEGPU_PROP_TIME_DOMAIN; prop <= ODEGPU_PROP_ACCESSORIES; ++prop) {
            if (!wants(copy_mode, prop)) continue;
            copy_rows(pool_array(p, prop), p->dims.problem_size, idx.d + count, 0, property_ptr(b, prop),
                      b->dims.batch_capacity, idx.d, 0, count, components_of(b->dims, prop), b->num_sms, b->stream);
        }
        CK(cudaStreamSynchronize(b->stream));
    });
}

int odegpu_device_pool_solve(odegpu_device_pool* p, const odegpu_model* model, const odegpu_solver_config* cfg,
                             const odegpu_ode_controls* ode, const odegpu_event_controls* ev,
                             odegpu_index batch_capacity, odegpu_index iterations, int32_t clustered) {
    return guarded([&] {
        check_pool(p);
        if (!model || !cfg || !ode) throw_invalid("null argument");
        if (iterations < 1) throw_invalid("solve_iteratively: iterations must be >= 1"); // solve.hpp:137
        if (batch_capacity < 1) throw_invalid("BatchDims: batch_capacity must be >= 1");
        const odegpu_system_dims sd = dims_of(*model);
        if (sd.system_dim != p->dims.system_dim || sd.param_count != p->dims.param_count ||
            sd.accessory_count != p->dims.accessory_count)
            throw_invalid("solve_pool: definition and pool dimensions disagree");
        const Index N = p->dims.problem_size;
        const Index cap = std::min<Index>(batch_capacity, N);
        // ODEGPU_POOL_TRACE=1: per-chunk timeline and host phases on stderr
        static const bool trace = std::getenv("ODEGPU_POOL_TRACE") != nullptr;
        const auto h0 = std::chrono::steady_clock::now();
        auto host_ms = [&] { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h0).count(); };
        DeviceGuard g(p->device);
        CK(cudaStreamSynchronize(p->stream));
        if (trace) std::fprintf(stderr, "[pool] host: entry sync %.3f ms\n", host_ms());
        // the working set: two batches (chunk k+1 gathers and launches while
        // chunk k's kernel drains, on another stream) and the permutation
        if (p->batch_cap != cap || p->batch_model.id != model->id || !p->batch[0]) {
            for (odegpu_batch*& b : p->batch) {
                if (b) odegpu_batch_destroy(b);
                b = nullptr;
            }
            const odegpu_batch_dims bd{cap, sd.system_dim, sd.param_count, sd.event_count, sd.accessory_count};
            for (odegpu_batch*& b : p->batch) b = batch_create(bd, p->device);
            p->batch_cap = cap;
            p->batch_model = *model;
        }
        // permutation: pool order, or longest first by the last solve's cost
        const std::size_t o_keys = align_up(std::size_t(N) * 4), o_iota = o_keys + align_up(std::size_t(N) * 4),
                          o_kout = o_iota + align_up(std::size_t(N) * 4), o_sorted = o_kout + align_up(std::size_t(N) * 4),
                          o_tmp = o_sorted + align_up(std::size_t(N) * 4);
        std::size_t tmp = 0;
        CK(cub::DeviceRadixSort::SortPairsDescending(nullptr, tmp, static_cast<unsigned*>(nullptr),
                                                      static_cast<unsigned*>(nullptr), static_cast<unsigned*>(nullptr),
                                                      static_cast<unsigned*>(nullptr), static_cast<int>(N), 0, 32,
                                                      p->stream));
        if (!p->order_block || p->order_bytes < o_tmp + tmp) {
            if (p->order_block) CK(cudaFree(p->order_block));
            p->order_block = nullptr;
            CK(cudaMalloc(&p->order_block, o_tmp + tmp));
            p->order_bytes = o_tmp + tmp;
        }
        auto* base = static_cast<unsigned char*>(p->order_block);
        auto* perm = reinterpret_cast<unsigned*>(base);
        auto* keys = reinterpret_cast<unsigned*>(base + o_keys);
        auto* iota = reinterpret_cast<unsigned*>(base + o_iota);
        auto* kout = reinterpret_cast<unsigned*>(base + o_kout);
        const int sms = p->batch[0]->num_sms;
        const int grid = static_cast<int>(std::max<Index>(1, std::min<Index>((N + 255) / 256, Index(sms) * 16)));
        const Index n_chunks = (N + cap - 1) / cap;
        const bool sorted = clustered && p->has_cost && N <= Index(0x7fffffff);
        if (sorted) {
            iota_kernel<<<grid, 256, 0, p->stream>>>(iota, N);
            CK(cudaGetLastError());
            CK(cudaMemcpyAsync(keys, p->cost, std::size_t(N) * 4, cudaMemcpyDeviceToDevice, p->stream));
            // longest first, then dealt round-robin into the chunks' rows (`perm`)
            auto* sorted_rows = reinterpret_cast<unsigned*>(base + o_sorted);
            CK(cub::DeviceRadixSort::SortPairsDescending(base + o_tmp, tmp, keys, kout, iota, sorted_rows,
                                                          static_cast<int>(N), 0, 32, p->stream));
            deal_kernel<<<grid, 256, 0, p->stream>>>(sorted_rows, N, n_chunks, perm);
            CK(cudaGetLastError());
        } else {
            iota_kernel<<<grid, 256, 0, p->stream>>>(perm, N);
            CK(cudaGetLastError());
        }
        // solve.hpp:159-161: any t1 < t0 in the pool and nothing is integrated
        unsigned long long* d_bad = nullptr;
        unsigned long long bad = ~0ull;
        CK(cudaMallocAsync(reinterpret_cast<void**>(&d_bad), sizeof bad, p->stream));
        CK(cudaMemsetAsync(d_bad, 0xff, sizeof bad, p->stream));
        pool_time_check_kernel<<<grid, 256, 0, p->stream>>>(p->td, N, d_bad);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(&bad, d_bad, sizeof bad, cudaMemcpyDeviceToHost, p->stream));
        CK(cudaFreeAsync(d_bad, p->stream));
        CK(cudaStreamSynchronize(p->stream));
        if (bad != ~0ull) throw_invalid("solve: system " + std::to_string(static_cast<long long>(bad)) + " has t1 < t0");
        if (trace) std::fprintf(stderr, "[pool] host: order + time check %.3f ms\n", host_ms());

        const dev::Controls c = prepare_solve(p->batch[0]->dims, model, cfg, ode, ev);
        const PoolOutcomes po{p->final_t, p->smallest, p->reason, p->accepted, p->rejected, p->detections,
                              p->secant_failures, p->cost};
        cudaEvent_t done[2] = {nullptr, nullptr};
        for (cudaEvent_t& e : done) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        struct Events {
            cudaEvent_t* e;
            ~Events() {
                for (int i = 0; i < 2; ++i)
                    if (e[i]) cudaEventDestroy(e[i]);
            }
        } guard{done};
        std::vector<cudaEvent_t> tev;
        auto mark = [&](cudaStream_t st) {
            if (!trace) return;
            cudaEvent_t e;
            CK(cudaEventCreate(&e));
            CK(cudaEventRecord(e, st));
            tev.push_back(e);
        };
        mark(p->stream);
        Index start = 0;
        for (Index k = 0; k < n_chunks; ++k) {
            odegpu_batch* b = p->batch[k & 1];
            mark(b->stream);
            // dealt chunks: N = q k + r, the first r hold q + 1 systems
            const Index n = sorted ? N / n_chunks + (k < N % n_chunks ? 1 : 0) : std::min(cap, N - start);
            const unsigned* rows = perm + start;
            // the batch's previous chunk is stored back before it is refilled
            // (its own stream orders that); the other batch's chunk may still run
            b->a.count = n;
            b->order_count = -1; // within a chunk: pool (permutation) order
            b->order_mode = ODEGPU_FETCH_NATURAL;
            for (int32_t prop = ODEGPU_PROP_TIME_DOMAIN; prop <= ODEGPU_PROP_ACCESSORIES; ++prop)
                copy_rows(property_ptr(b, prop), cap, static_cast<const unsigned*>(nullptr), 0, pool_array(p, prop), N,
                          rows, 0, n, components_of(b->dims, prop), sms, b->stream);
            launch_reset_outcomes(b, 0, n); // linear_set(All) of the chunk resets its outcomes (batch.cpp:102-103)
            for (Index it = 0; it < iterations;) {
                enqueue_time_check(b);
                b->fuse_request = iterations - it;
                b->build_order = false;
                launch_model(b, *model, cfg->algorithm, c);
                it += b->fused_done;
            }
            // end points and outcomes back into the pool rows (params never change)
            for (int32_t prop : {ODEGPU_PROP_TIME_DOMAIN, ODEGPU_PROP_STATE, ODEGPU_PROP_ACCESSORIES})
                copy_rows(pool_array(p, prop), N, rows, 0, property_ptr(b, prop), cap,
                          static_cast<const unsigned*>(nullptr), 0, n, components_of(b->dims, prop), sms, b->stream);
            const int og = static_cast<int>(std::max<Index>(1, std::min<Index>((n + 255) / 256, Index(sms) * 8)));
            store_outcomes_kernel<unsigned><<<og, 256, 0, b->stream>>>(b->a, n, rows, 0, po);
            CK(cudaGetLastError());
            CK(cudaEventRecord(done[k & 1], b->stream));
            mark(b->stream);
            start += n;
        }
        if (trace) std::fprintf(stderr, "[pool] host: chunks enqueued %.3f ms\n", host_ms());
        for (odegpu_batch* b : p->batch) CK(cudaStreamSynchronize(b->stream));
        if (trace) std::fprintf(stderr, "[pool] host: done %.3f ms\n", host_ms());
        if (trace) {
            for (std::size_t i = 1; i + 1 < tev.size(); i += 2) {
                float a = 0, d = 0;
                cudaEventElapsedTime(&a, tev[0], tev[i]);
                cudaEventElapsedTime(&d, tev[i], tev[i + 1]);
                std::fprintf(stderr, "[pool] chunk %zu: start %.3f ms, gather+solve+store %.3f ms\n", i / 2, a, d);
            }
            for (auto e : tev) cudaEventDestroy(e);
        }
        p->has_cost = true;
    });
}

} // extern "C"
