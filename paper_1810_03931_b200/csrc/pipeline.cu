// pipeline.cu — chunked problem-pool batching (the device side of
// src/scan.cpp:88-112 run_chunks) with double-buffered H2D/D2H on two
// streams, and its multi-GPU form (one host thread and one contiguous slice
// per device; no inter-GPU traffic: systems are independent).
#include <cuda.h> // stream memory operation types only (entry points via cudaGetDriverEntryPoint)
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <map>
#include <mutex>
#include <span>
#include <string>
#include <thread>
#include <vector>

#include "internal.cuh"

using namespace odegpu;
using namespace odegpu::detail;

namespace odegpu::detail {

namespace {
/// Process-wide cache of page-locked host blocks. Pinning is slow (the
/// driver locks every page: ~100 ms for the ~170 MB of staging a 2^16-system
/// scan pipeline holds, and about as long to unpin), and scan drivers create
/// a pipeline per scan: freed blocks are kept (up to ODEGPU_PINNED_CACHE_MB,
/// default 2048) and handed out again for requests of up to their size.
struct PinnedCache {
    std::mutex mu;
    std::multimap<size_t, void*> free_blocks; // size -> block
    std::map<void*, size_t> sizes;            // every block this cache allocated
    size_t cached = 0;
    size_t limit = [] {
        const char* e = std::getenv("ODEGPU_PINNED_CACHE_MB");
        return (e ? size_t(std::max(0, std::atoi(e))) : size_t(2048)) << 20;
    }();
};
PinnedCache& pinned_cache() {
    static PinnedCache* c = new PinnedCache; // never destroyed: blocks may be freed during exit
    return *c;
}
} // namespace

void* host_alloc(size_t bytes) {
    if (bytes == 0) return nullptr;
    PinnedCache& c = pinned_cache();
    {
        std::lock_guard<std::mutex> lock(c.mu);
        auto it = c.free_blocks.lower_bound(bytes);
        if (it != c.free_blocks.end() && it->first <= bytes + bytes / 4) { // reuse a block of up to 1.25x
            void* q = it->second;
            c.cached -= it->first;
            c.free_blocks.erase(it);
            return q;
        }
    }
    void* q = nullptr;
    CK(cudaMallocHost(&q, bytes));
    std::lock_guard<std::mutex> lock(c.mu);
    c.sizes[q] = bytes;
    return q;
}

void host_free(void* q) {
    if (!q) return;
    PinnedCache& c = pinned_cache();
    std::lock_guard<std::mutex> lock(c.mu);
    const auto it = c.sizes.find(q);
    if (it == c.sizes.end()) {
        cudaFreeHost(q);
        return;
    }
    if (c.cached + it->second <= c.limit) {
        c.free_blocks.emplace(it->second, q);
        c.cached += it->second;
    } else {
        c.sizes.erase(it);
        cudaFreeHost(q);
    }
}

void OutcomeStage::allocate(Index cap) {
    const size_t n = size_t(cap);
    const size_t bytes = n * (8 * 6 + 1) + 64;
    block = host_alloc(bytes);
    char* p = static_cast<char*>(block);
    final_t = reinterpret_cast<double*>(p);
    smallest = final_t + n;
    accepted = reinterpret_cast<Index*>(smallest + n);
    rejected = accepted + n;
    detections = rejected + n;
    secant_failures = detections + n;
    reason = reinterpret_cast<std::uint8_t*>(secant_failures + n);
}

void OutcomeStage::release() {
    host_free(block);
    block = nullptr;
}

void OutcomeStage::fetch(const odegpu_batch* b, Index start, Index count, cudaStream_t s) {
    const size_t n = size_t(count);
    CK(cudaMemcpyAsync(final_t, b->a.final_t + start, n * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(smallest, b->a.smallest_step + start, n * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(accepted, b->a.accepted + start, n * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(rejected, b->a.rejected + start, n * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(detections, b->a.detections + start, n * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(secant_failures, b->a.secant_failures + start, n * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(reason, b->a.reason + start, n, cudaMemcpyDeviceToHost, s));
}

void OutcomeStage::pack(odegpu_outcome* out, Index count) const {
    for (Index i = 0; i < count; ++i) {
        odegpu_outcome o{};
        o.final_t = final_t[i];
        o.reason = reason[i];
        o.accepted_steps = accepted[i];
        o.rejected_steps = rejected[i];
        o.event_detections = detections[i];
        o.secant_failures = secant_failures[i];
        o.smallest_step = smallest[i];
        out[i] = o;
    }
}

void download_outcomes(odegpu_batch* b, Index start, Index count, odegpu_outcome* host) {
    if (!b->out_stage) { // pinned staging, kept for the batch's lifetime
        auto* st = new OutcomeStage;
        try {
            st->allocate(b->dims.batch_capacity);
        } catch (...) {
            delete st;
            throw;
        }
        b->out_stage = st;
    }
    auto* st = static_cast<OutcomeStage*>(b->out_stage);
    st->fetch(b, start, count, b->stream);
    CK(cudaStreamSynchronize(b->stream));
    st->pack(host, count);
}

void release_batch_stage(odegpu_batch* b) {
    if (!b->out_stage) return;
    auto* st = static_cast<OutcomeStage*>(b->out_stage);
    st->release();
    delete st;
    b->out_stage = nullptr;
}

namespace {

// AoS odensemble::SystemOutcome records (56 B) from the SoA outcome fields,
// so one D2H lands them in the caller's array without host-side packing.
__global__ void pack_outcomes_kernel(dev::BatchArrays b, Index count, odegpu_outcome* dst) {
    for (Index i = blockIdx.x * static_cast<Index>(blockDim.x) + threadIdx.x; i < count;
         i += static_cast<Index>(gridDim.x) * blockDim.x) {
        odegpu_outcome o{};
        o.final_t = b.final_t[i];
        o.reason = b.reason[i];
        o.accepted_steps = b.accepted[i];
        o.rejected_steps = b.rejected[i];
        o.event_detections = b.detections[i];
        o.secant_failures = b.secant_failures[i];
        o.smallest_step = b.smallest_step[i];
        dst[i] = o;
    }
}

bool is_pinned(const void* p) {
    if (!p) return false;
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

double* pinned(Index doubles) {
    return doubles > 0 ? static_cast<double*>(host_alloc(size_t(doubles) * 8)) : nullptr;
}

/// One half of the double buffer: a device batch plus pinned staging.
struct Slot {
    odegpu_batch* batch = nullptr; // compute runs on batch->stream
    cudaEvent_t loaded = nullptr;   // H2D of the slot's chunk done (copy-in stream)
    cudaEvent_t computed = nullptr; // kernels of the chunk done (compute stream)
    cudaEvent_t done = nullptr;     // D2H of the chunk done (copy-out stream)
    double* fin_td = nullptr; // endpoints of the chunk, [comps][cap]
    double* fin_y = nullptr;
    double* fin_acc = nullptr;
    odegpu_outcome* d_packed = nullptr;   // device AoS outcome records [cap]
    odegpu_outcome* fin_out = nullptr;    // pinned AoS staging [cap]
    double* rec_td = nullptr; // recorded iterations, [n_rec][comps][cap]
    double* rec_y = nullptr;
    double* rec_acc = nullptr;
    std::vector<OutcomeStage> rec_out;
    Index start = 0, count = 0;
    bool busy = false;
};

/// The streaming mode's device state (odegpu_pipeline_mode STREAMING): one
/// batch holding the whole pool, the chunk gate and the packed records.
constexpr cuuint32_t kStreamAbortHost = 0x80000000u; // dev::kStreamAbort

struct StreamState {
    static constexpr Index kMaxGranules = 256;
    odegpu_batch* batch = nullptr;
    Index cap = 0;
    unsigned* gate = nullptr;               // [0] chunks landed, [1 + c] systems of chunk c finished
    unsigned long long* bad = nullptr;      // StreamGate::bad (4 words)
    unsigned long long* h_bad = nullptr;    // pinned mirror
    unsigned short* group_of = nullptr;     // [kMaxGranules] granule -> copy-out group (device)
    unsigned short* h_group_of = nullptr;   // pinned staging
    unsigned char* packed = nullptr;        // [cap] x 56 B
    cudaEvent_t prologue = nullptr;
    void release() {
        if (batch) {
            cudaStreamSynchronize(batch->stream);
            odegpu_batch_destroy(batch);
        }
        for (void* q : {static_cast<void*>(gate), static_cast<void*>(bad), static_cast<void*>(packed)})
            if (q) cudaFree(q);
        if (h_bad) cudaFreeHost(h_bad);
        if (group_of) cudaFree(group_of);
        if (h_group_of) cudaFreeHost(h_group_of);
        if (prologue) cudaEventDestroy(prologue);
        *this = StreamState{};
    }
};

struct Run {
    const odegpu_pool_view* pool;
    const odegpu_pool_out* out;
    const odegpu_solver_config* cfg;
    const odegpu_ode_controls* ode;
    const odegpu_event_controls* ev;
    Index iterations, record_from;
    uint32_t mask;
    odegpu_chunk_sink sink;
    void* user;
    std::mutex* sink_mutex; // serialises sinks across device threads
    odegpu_scan_tally* tally = nullptr; // scan tallies, merged under sink_mutex
};

} // namespace
} // namespace odegpu::detail

/// The pipeline object: everything a chunked run needs, allocated once.
struct odegpu_pipeline {
    odegpu_model model{};
    odegpu_system_dims sd{};
    Index cap = 0;
    int device = 0;
    Index rec_capacity = 0; // recorded iterations the staging can hold
    // chunks in flight (device batches + pinned staging): copy-in, compute
    // (two), copy-out and the ones whose H2D runs ahead. 6 measured best on
    // one B200 (e2e, bench chunking: cfg2 3.06 ms vs 3.19 with 4 and 3.09
    // with 8; cfg1 / cfg4 / cfg5 flat); ODEGPU_PIPELINE_SLOTS overrides it
    static constexpr int kMaxSlots = 8;
    int n_slots = 6;
    odegpu::detail::Slot slots[kMaxSlots];
    cudaStream_t copy_in = nullptr, copy_out = nullptr;
    std::vector<odegpu_outcome> packed;
    unsigned long long* d_tally = nullptr; // device scan tally (kTallySlots counters)
    unsigned long long* h_tally = nullptr; // pinned mirror
    int32_t mode = ODEGPU_PIPELINE_AUTO;      // odegpu_pipeline_set_mode
    int32_t last_mode = ODEGPU_PIPELINE_AUTO; // what the last run used
    odegpu::detail::StreamState stream;       // streaming mode, allocated on first use

    ~odegpu_pipeline() {
        stream.release();
        // no copy may still target a staging block once it is back in the
        // pinned cache (host_free), so the copy streams drain first
        for (cudaStream_t st : {copy_in, copy_out})
            if (st) cudaStreamSynchronize(st);
        for (auto& s : slots) {
            if (s.batch) {
                cudaStreamSynchronize(s.batch->stream);
                odegpu_batch_destroy(s.batch);
            }
            for (cudaEvent_t e : {s.loaded, s.computed, s.done})
                if (e) cudaEventDestroy(e);
            for (double* p : {s.fin_td, s.fin_y, s.fin_acc, s.rec_td, s.rec_y, s.rec_acc})
                odegpu::detail::host_free(p);
            odegpu::detail::host_free(s.fin_out);
            if (s.d_packed) cudaFree(s.d_packed);
            for (auto& o : s.rec_out) o.release();
        }
        for (cudaStream_t st : {copy_in, copy_out})
            if (st) {
                cudaStreamSynchronize(st);
                cudaStreamDestroy(st);
            }
        if (d_tally) cudaFree(d_tally);
        odegpu::detail::host_free(h_tally);
    }
};

namespace odegpu::detail {
namespace {

odegpu_pipeline* pipeline_create(const odegpu_model& model, Index capacity, int device) {
    if (capacity < 1) throw_invalid("BatchDims: batch_capacity must be >= 1");
    auto* p = new odegpu_pipeline;
    try {
        p->model = model;
        p->sd = dims_of(model);
        p->cap = capacity;
        p->device = device;
        if (const char* e = std::getenv("ODEGPU_PIPELINE_SLOTS"))
            p->n_slots = std::clamp(std::atoi(e), 3, odegpu_pipeline::kMaxSlots);
        DeviceGuard g(device);
        const auto& sd = p->sd;
        const odegpu_batch_dims bd{capacity, sd.system_dim, sd.param_count, sd.event_count, sd.accessory_count};
        CK(cudaStreamCreateWithFlags(&p->copy_in, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&p->copy_out, cudaStreamNonBlocking));
        for (auto& s : std::span(p->slots, size_t(p->n_slots))) {
            s.batch = batch_create(bd, device);
            for (cudaEvent_t* e : {&s.loaded, &s.computed, &s.done})
                CK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
            // endpoint staging (fin_*) is allocated by the first run that
            // writes back into pageable arrays (ensure_endpoint_staging)
            CK(cudaMalloc(&s.d_packed, size_t(capacity) * sizeof(odegpu_outcome)));
        }
        CK(cudaMalloc(&p->d_tally, dev::kTallySlots * sizeof(unsigned long long)));
        p->h_tally = static_cast<unsigned long long*>(host_alloc(dev::kTallySlots * sizeof(unsigned long long)));
    } catch (...) {
        delete p;
        throw;
    }
    return p;
}

/// Pinned staging for endpoints written back into pageable arrays, in the
/// first `slots` slots, allocated when a run first needs it.
void ensure_endpoint_staging(odegpu_pipeline* p, int slots, bool td, bool y, bool acc, bool out) {
    const auto& sd = p->sd;
    const Index cap = p->cap;
    for (auto& s : std::span(p->slots, size_t(slots))) {
        if (td && !s.fin_td) s.fin_td = pinned(2 * cap);
        if (y && !s.fin_y) s.fin_y = pinned(sd.system_dim * cap);
        if (acc && sd.accessory_count && !s.fin_acc) s.fin_acc = pinned(sd.accessory_count * cap);
        if (out && !s.fin_out) s.fin_out = static_cast<odegpu_outcome*>(host_alloc(size_t(cap) * sizeof(odegpu_outcome)));
    }
}

/// Grow the recorded-iteration staging to n_rec iterations (first `slots` slots).
void reserve_records(odegpu_pipeline* p, int slots, Index n_rec, uint32_t mask) {
    if (n_rec <= p->rec_capacity) return;
    const auto& sd = p->sd;
    const Index cap = p->cap;
    for (auto& s : std::span(p->slots, size_t(slots))) {
        for (double* q : {s.rec_td, s.rec_y, s.rec_acc})
            host_free(q);
        s.rec_td = s.rec_y = s.rec_acc = nullptr;
        for (auto& o : s.rec_out) o.release();
        s.rec_out.clear();
        if (mask & 1u) s.rec_td = pinned(n_rec * 2 * cap);
        if (mask & 2u) s.rec_y = pinned(n_rec * sd.system_dim * cap);
        if (mask & 8u) s.rec_acc = pinned(n_rec * sd.accessory_count * cap);
        if (mask & 16u) {
            s.rec_out.resize(size_t(n_rec));
            for (auto& o : s.rec_out) o.allocate(cap);
        }
    }
    p->rec_capacity = n_rec;
    p->packed.resize(size_t(n_rec * cap));
}

/// Where a pipeline takes its chunks from: consecutive chunks of one range
/// (a single device), or a queue shared by every device of a multi-GPU run —
/// each device thread claims the next chunk with fetch_add, the cross-device
/// analogue of the reference's worker tile claim (solve.hpp:94-95), so fast
/// devices (or devices that drew cheap systems) take more chunks.
struct ChunkSource {
    std::atomic<Index>* shared = nullptr; // multi-device queue (chunk starts), or
    Index next = 0;                       // the private cursor of a single range
    Index end = 0;
    Index step = 0;
    /// [start, start + count) of the next chunk; false when drained.
    bool claim(Index cap, Index* start, Index* count) {
        const Index s = shared ? shared->fetch_add(step) : next;
        if (!shared) next += step;
        if (s >= end) return false;
        *start = s;
        *count = std::min(cap, end - s);
        return true;
    }
};

/// Runs the chunks `src` hands out through the pipeline's device.
void run_chunks(odegpu_pipeline* p, const Run& j, ChunkSource& src) {
    const odegpu_pool_dims& pd = j.pool->dims;
    const odegpu_system_dims& sd = p->sd;
    if (sd.system_dim != pd.system_dim || sd.param_count != pd.param_count ||
        sd.accessory_count != pd.accessory_count)
        throw_invalid("solve_pool: definition and pool dimensions disagree");
    const Index cap = p->cap;
    const odegpu_batch_dims bd{cap, sd.system_dim, sd.param_count, sd.event_count, sd.accessory_count};
    const dev::Controls c = prepare_solve(bd, &p->model, j.cfg, j.ode, j.ev);
    const Index n_rec = j.sink ? j.iterations - j.record_from : 0;
    const uint32_t mask = j.sink ? j.mask : 0u;
    const Index N = pd.problem_size;
    const bool r_td = mask & 1u, r_y = mask & 2u, r_acc = (mask & 8u) && sd.accessory_count, r_out = mask & 16u;
    DeviceGuard g(p->device);
    unsigned long long* tally = j.tally ? p->d_tally : nullptr;
    // zeroed on the copy-in stream: every chunk's kernels wait for its H2D
    if (tally) CK(cudaMemsetAsync(tally, 0, dev::kTallySlots * sizeof(unsigned long long), p->copy_in));
    for (auto& s : std::span(p->slots, size_t(p->n_slots))) s.batch->a.tally = tally;
    // Slots in flight: all of them for a plain run; 3 for a run that records
    // iterations (a scan): every chunk's records go through the host sink
    // anyway, and each slot holds n_rec iterations of pinned staging
    const int kSlots = n_rec > 0 ? std::min(p->n_slots, 3) : p->n_slots;
    if (n_rec > 0) {
        // (re)allocate when the mask needs arrays the staging lacks
        const Slot& s0 = p->slots[0];
        const bool lacking = (r_td && !s0.rec_td) || (r_y && !s0.rec_y) || (r_acc && !s0.rec_acc) ||
                             (r_out && s0.rec_out.empty());
        if (lacking) p->rec_capacity = 0;
        reserve_records(p, kSlots, n_rec, mask);
    }

    // Endpoint write-back: straight into the caller's arrays when they are
    // page-locked (async D2H, no host copy), else via pinned staging.
    const odegpu_pool_out none{};
    const odegpu_pool_out& o = j.out ? *j.out : none;
    // Time domains a solve cannot change (hooks.hpp kKeepsTimeDomain) need
    // no copy back into the pool array they were read from (in-place runs).
    const bool td_back = o.time_domain && !(o.time_domain == j.pool->time_domain && keeps_time_domain(p->model));
    const bool d_td = is_pinned(o.time_domain), d_y = is_pinned(o.state),
               d_acc = sd.accessory_count && is_pinned(o.accessories), d_out = is_pinned(o.outcomes);
    ensure_endpoint_staging(p, kSlots, td_back && !d_td, o.state && !d_y, o.accessories && !d_acc,
                            o.outcomes && !d_out);

    // Consume a finished slot: validation flag, staged write-back, sink.
    auto drain = [&](Slot& s) {
        if (!s.busy) return;
        CK(cudaEventSynchronize(s.done));
        s.busy = false;
        if (*s.batch->host_flag != ~0ull)
            throw_invalid("solve: system " + std::to_string(static_cast<long long>(*s.batch->host_flag)) +
                          " has t1 < t0");
        const Index n = s.count, off = s.start;
        auto put = [&](double* dst, const double* src, Index comps) {
            for (Index cc = 0; cc < comps; ++cc) std::memcpy(dst + off + cc * N, src + cc * cap, size_t(n) * 8);
        };
        if (td_back && !d_td) put(o.time_domain, s.fin_td, 2);
        if (o.state && !d_y) put(o.state, s.fin_y, sd.system_dim);
        if (o.accessories && sd.accessory_count && !d_acc) put(o.accessories, s.fin_acc, sd.accessory_count);
        if (o.outcomes && !d_out) std::memcpy(o.outcomes + off, s.fin_out, size_t(n) * sizeof(odegpu_outcome));
        if (j.sink) { // also with no recorded iteration (n_rec = 0): the chunk is done
            if (r_out)
                for (Index r = 0; r < n_rec; ++r) s.rec_out[size_t(r)].pack(p->packed.data() + r * n, n);
            // compact the recorded arrays from stride cap to stride n
            auto compact = [&](double* q, Index comps) {
                if (!q || n == cap) return;
                for (Index r = 0; r < n_rec; ++r)
                    for (Index cc = 0; cc < comps; ++cc)
                        std::memmove(q + (r * comps + cc) * n, q + (r * comps + cc) * cap, size_t(n) * 8);
            };
            if (r_td) compact(s.rec_td, 2);
            if (r_y) compact(s.rec_y, sd.system_dim);
            if (r_acc) compact(s.rec_acc, sd.accessory_count);
            const odegpu_chunk_record rec{r_td ? s.rec_td : nullptr, r_y ? s.rec_y : nullptr,
                                          r_acc ? s.rec_acc : nullptr, r_out ? p->packed.data() : nullptr};
            int rc;
            {
                std::lock_guard<std::mutex> lock(*j.sink_mutex);
                rc = j.sink(off, n, n_rec, &rec, j.user);
            }
            if (rc != 0) throw Error(rc, "solve_pool: chunk sink returned " + std::to_string(rc));
        }
    };

    // ODEGPU_PIPELINE_TRACE=1: per-chunk CUDA-event timeline on stderr
    static const bool trace = std::getenv("ODEGPU_PIPELINE_TRACE") != nullptr;
    std::vector<cudaEvent_t> tev;
    auto mark = [&](cudaStream_t st) {
        if (!trace) return;
        cudaEvent_t e;
        CK(cudaEventCreate(&e));
        CK(cudaEventRecord(e, st));
        tev.push_back(e);
    };
    // Three-stage pipeline over n_slots device batches: chunk k's H2D runs on
    // the copy-in stream, its kernels on the slot batch's stream (after the
    // H2D event), its D2H on the copy-out stream (after the kernels' event),
    // so H2D(k+1), the kernels of k and D2H(k-1) overlap (PCIe is full
    // duplex: 55 GB/s each way measured on the B200 box, 99 GB/s both). A
    // slot is refilled only after its previous chunk was drained on the host.
    int k = 0;
    try {
        Index start = 0, n = 0;
        for (; src.claim(cap, &start, &n); ++k) {
            Slot& s = p->slots[k % kSlots];
            drain(s); // the slot's previous chunk must be consumed before reuse
            odegpu_batch* b = s.batch;
            mark(p->copy_in);
            s.start = start;
            s.count = n;
            b->a.count = n;
            b->order_count = -1; // new systems: no cost order until this chunk's first solve
            // linear_set(All) of the chunk: pool -> batch (batch.cpp:78-104), on the copy-in stream
            copy_h2d_strided(b->a.td, cap, 0, j.pool->time_domain, N, start, n, 2, p->copy_in);
            copy_h2d_strided(b->a.state, cap, 0, j.pool->state, N, start, n, sd.system_dim, p->copy_in);
            if (sd.param_count)
                copy_h2d_strided(const_cast<Real*>(b->a.params), cap, 0, j.pool->parameters, N, start, n,
                                 sd.param_count, p->copy_in);
            if (sd.accessory_count)
                copy_h2d_strided(b->a.acc, cap, 0, j.pool->accessories, N, start, n, sd.accessory_count, p->copy_in);
            CK(cudaEventRecord(s.loaded, p->copy_in));
            // kernels: fresh outcomes, then every iteration back to back.
            // At most two chunks compute at once: chunk k starts once chunk
            // k-2's kernels are done, so chunk k-1 has the device to itself
            // but for chunk k filling its tail. (With every in-flight chunk
            // computing at once they all finished together, late: their D2H,
            // and so the next chunks' H2D into the freed slots, came in
            // bursts that left the device idle between them — 4-chunk groups
            // in the ODEGPU_PIPELINE_TRACE timeline of the 2^24 pool.)
            CK(cudaStreamWaitEvent(b->stream, s.loaded, 0));
            if (k >= 2) CK(cudaStreamWaitEvent(b->stream, p->slots[(k - 2) % kSlots].computed, 0));
            mark(b->stream);
            launch_reset_outcomes(b, 0, n);
            // no per-iteration tally or snapshot to take: the iterations may
            // run fused in one launch (solve_iteratively without a sink)
            const bool fuse = !tally && n_rec == 0;
            for (Index it = 0; it < j.iterations;) {
                enqueue_time_check(b);
                b->fuse_request = fuse ? j.iterations - it : 1;
                b->build_order = it + b->fuse_request < j.iterations; // the chunk's last solve: order unused
                launch_model(b, p->model, j.cfg->algorithm, c);
                const Index done = b->fused_done;
                it += done;
                if (done > 1) continue; // fused: no per-iteration work below
                if (tally) launch_tally(b, tally, false);
                if (n_rec > 0 && it - 1 >= j.record_from) { // snapshots stay ordered with the kernels
                    const Index r = it - 1 - j.record_from;
                    if (r_td) copy_d2h_strided(s.rec_td + r * 2 * cap, cap, 0, b->a.td, cap, 0, n, 2, b->stream);
                    if (r_y)
                        copy_d2h_strided(s.rec_y + r * sd.system_dim * cap, cap, 0, b->a.state, cap, 0, n,
                                         sd.system_dim, b->stream);
                    if (r_acc)
                        copy_d2h_strided(s.rec_acc + r * sd.accessory_count * cap, cap, 0, b->a.acc, cap, 0, n,
                                         sd.accessory_count, b->stream);
                    if (r_out) s.rec_out[size_t(r)].fetch(b, 0, n, b->stream);
                }
            }
            if (tally) launch_tally(b, tally, true);
            if (o.outcomes) {
                pack_outcomes_kernel<<<grid_for(b, n, 256), 256, 0, b->stream>>>(b->a, n, s.d_packed);
                CK(cudaGetLastError());
                ++b->launches;
            }
            mark(b->stream);
            CK(cudaEventRecord(s.computed, b->stream));
            // endpoints on the copy-out stream
            CK(cudaStreamWaitEvent(p->copy_out, s.computed, 0));
            mark(p->copy_out);
            cudaStream_t out_s = p->copy_out;
            if (td_back) {
                if (d_td) copy_d2h_strided(o.time_domain, N, start, b->a.td, cap, 0, n, 2, out_s);
                else copy_d2h_strided(s.fin_td, cap, 0, b->a.td, cap, 0, n, 2, out_s);
            }
            if (o.state) {
                if (d_y) copy_d2h_strided(o.state, N, start, b->a.state, cap, 0, n, sd.system_dim, out_s);
                else copy_d2h_strided(s.fin_y, cap, 0, b->a.state, cap, 0, n, sd.system_dim, out_s);
            }
            if (o.accessories && sd.accessory_count) {
                if (d_acc)
                    copy_d2h_strided(o.accessories, N, start, b->a.acc, cap, 0, n, sd.accessory_count, out_s);
                else
                    copy_d2h_strided(s.fin_acc, cap, 0, b->a.acc, cap, 0, n, sd.accessory_count, out_s);
            }
            if (o.outcomes)
                CK(cudaMemcpyAsync(d_out ? o.outcomes + start : s.fin_out, s.d_packed,
                                   size_t(n) * sizeof(odegpu_outcome), cudaMemcpyDeviceToHost, out_s));
            CK(cudaMemcpyAsync(b->host_flag, b->first_bad, sizeof(unsigned long long), cudaMemcpyDeviceToHost, out_s));
            mark(out_s);
            CK(cudaEventRecord(s.done, out_s));
            s.busy = true;
        }
        for (int r = 0; r < kSlots; ++r) drain(p->slots[(k + r) % kSlots]); // oldest first
        if (trace && !tev.empty()) {
            for (size_t c = 0; c + 4 < tev.size(); c += 5) {
                float a = 0, h = 0, x = 0, w = 0, d = 0;
                cudaEventElapsedTime(&a, tev[0], tev[c]);
                cudaEventElapsedTime(&h, tev[c], tev[c + 1]);
                cudaEventElapsedTime(&x, tev[c + 1], tev[c + 2]);
                cudaEventElapsedTime(&w, tev[c + 2], tev[c + 3]);
                cudaEventElapsedTime(&d, tev[c + 3], tev[c + 4]);
                std::fprintf(stderr,
                             "[pipeline] chunk %zu: h2d at %.3f ms, +%.3f to kernels, kernels %.3f, +%.3f to d2h, "
                             "d2h %.3f\n",
                             c / 5, a, h, x, w, d);
            }
            for (auto e : tev) cudaEventDestroy(e);
        }
        if (tally) { // both slot streams are drained: merge the device tally
            CK(cudaMemcpy(p->h_tally, tally, dev::kTallySlots * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
            const unsigned long long* h = p->h_tally;
            std::lock_guard<std::mutex> lock(*j.sink_mutex);
            odegpu_scan_tally& t = *j.tally;
            for (int r = 0; r < 4; ++r) t.reason_counts[r] += Index(h[dev::kTallyReason0 + r]);
            t.secant_failures += Index(h[dev::kTallySecantFailures]);
            t.detections += Index(h[dev::kTallyDetections]);
            t.detections_outside_zone += Index(h[dev::kTallyOutsideZone]);
            double mr = 0;
            std::memcpy(&mr, h + dev::kTallyMaxRatio, sizeof mr);
            t.max_residual_ratio = std::max(t.max_residual_ratio, mr);
            t.start_time_not_advanced += Index(h[dev::kTallyStartNotAdvanced]);
            t.nonfinite_systems += Index(h[dev::kTallyNonfinite]);
        }
        for (auto& s : std::span(p->slots, size_t(p->n_slots))) s.batch->a.tally = nullptr;
    } catch (...) {
        // Quiesce every stream of the pipeline before handing control back:
        // queued D2H copies could otherwise still write into the caller's
        // page-locked arrays after the error returns, and a later run could
        // reuse a slot whose old copies are pending.
        for (auto& s : std::span(p->slots, size_t(p->n_slots))) s.batch->a.tally = nullptr;
        cudaStreamSynchronize(p->copy_in);
        for (auto& s : std::span(p->slots, size_t(p->n_slots)))
            if (s.batch) cudaStreamSynchronize(s.batch->stream);
        cudaStreamSynchronize(p->copy_out);
        for (auto& s : std::span(p->slots, size_t(p->n_slots))) s.busy = false;
        throw;
    }
}

// ---------------------------------------------------------------- streaming

using WriteValueFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
using WaitValueFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

/// cuStreamWriteValue32 / cuStreamWaitValue32 from the driver the runtime
/// runs on (no link-time dependency on libcuda); null when unavailable.
struct StreamMemOps {
    WriteValueFn write = nullptr;
    WaitValueFn wait = nullptr;
};

const StreamMemOps& stream_memops() {
    static const StreamMemOps ops = [] {
        StreamMemOps o;
        void* w = nullptr;
        void* v = nullptr;
        cudaDriverEntryPointQueryResult q1{}, q2{};
        if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &w, cudaEnableDefault, &q1) == cudaSuccess &&
            cudaGetDriverEntryPoint("cuStreamWaitValue32", &v, cudaEnableDefault, &q2) == cudaSuccess &&
            q1 == cudaDriverEntryPointSuccess && q2 == cudaDriverEntryPointSuccess && w && v) {
            o.write = reinterpret_cast<WriteValueFn>(w);
            o.wait = reinterpret_cast<WaitValueFn>(v);
        }
        cudaGetLastError();
        return o;
    }();
    return ops;
}

void check_cu(CUresult r, const char* what) {
    if (r != CUDA_SUCCESS) throw Error(ODEGPU_ERR_CUDA, std::string(what) + ": CUresult " + std::to_string(int(r)));
}

/// Device bytes per system of the streaming batch and its side arrays.
Index stream_bytes_per_system(const odegpu_system_dims& sd) {
    return 8 * (2 + sd.system_dim + sd.param_count + sd.accessory_count) + 49 + 56 + 4 + 16;
}

/// Why the streaming mode does not apply to this run (nullptr: it does).
const char* stream_blocker(odegpu_pipeline* p, const Run& j) {
    if (j.sink || j.tally) return "a chunk sink or scan tally needs per-chunk iterations";
    if (j.iterations > 1 && !fusable_iterations(p->model)) return "the model's iterations do not fuse";
    if (j.iterations > 65535) return "more than 65535 fused iterations";
    const Index N = j.pool->dims.problem_size;
    if (N >= (Index(1) << 31)) return "pool too large for 32-bit system indices";
    const odegpu_system_dims& sd = p->sd;
    if (!is_pinned(j.pool->time_domain) || !is_pinned(j.pool->state) ||
        (sd.param_count && !is_pinned(j.pool->parameters)) || (sd.accessory_count && !is_pinned(j.pool->accessories)))
        return "pool arrays are not page-locked";
    if (j.out) {
        const odegpu_pool_out& o = *j.out;
        if ((o.time_domain && !is_pinned(o.time_domain)) || (o.state && !is_pinned(o.state)) ||
            (o.accessories && sd.accessory_count && !is_pinned(o.accessories)) ||
            (o.outcomes && !is_pinned(o.outcomes)))
            return "out arrays are not page-locked";
    }
    const StreamMemOps& ops = stream_memops();
    if (!ops.write || !ops.wait) return "stream memory operations unavailable";
    if (p->stream.cap < N) {
        size_t free_b = 0, total_b = 0;
        DeviceGuard g(p->device);
        CK(cudaMemGetInfo(&free_b, &total_b));
        const double have = double(free_b) + (p->stream.batch ? double(p->stream.cap) * double(stream_bytes_per_system(sd)) : 0.0);
        if (double(N) * double(stream_bytes_per_system(sd)) > 0.6 * have) return "pool does not fit the device";
    }
    return nullptr;
}

/// (Re)allocates the streaming state for N systems.
void stream_reserve(odegpu_pipeline* p, Index N) {
    StreamState& st = p->stream;
    if (st.batch && st.cap >= N) return;
    st.release();
    DeviceGuard g(p->device);
    const auto& sd = p->sd;
    const odegpu_batch_dims bd{N, sd.system_dim, sd.param_count, sd.event_count, sd.accessory_count};
    try {
        st.batch = batch_create(bd, p->device);
        st.cap = N;
        CK(cudaMalloc(&st.gate, sizeof(unsigned) * (1 + StreamState::kMaxGranules)));
        CK(cudaMalloc(&st.bad, 4 * sizeof(unsigned long long)));
        CK(cudaMallocHost(&st.h_bad, 4 * sizeof(unsigned long long)));
        CK(cudaMalloc(&st.group_of, sizeof(unsigned short) * StreamState::kMaxGranules));
        CK(cudaMallocHost(&st.h_group_of, sizeof(unsigned short) * StreamState::kMaxGranules));
        CK(cudaMalloc(&st.packed, 56 * size_t(N)));
        CK(cudaEventCreateWithFlags(&st.prologue, cudaEventDisableTiming));
    } catch (...) {
        st.release();
        throw;
    }
}

/// log2 of the systems per granule of a streamed pool: N/256 rounded up to
/// a power of two, at least 4096 (cfg2's 2^20 pool: 16 Ki systems, 1.3 MB
/// of inputs) and 32 — every 128-byte line of every SoA array lies in one
/// granule, and a lane finds its granule with a shift. ODEGPU_STREAM_CHUNK
/// overrides the size (tuning; rounded up to a power of two).
unsigned stream_granule_shift(Index N) {
    Index s = std::max<Index>((N + StreamState::kMaxGranules - 1) / StreamState::kMaxGranules, 4096);
    if (const char* e = std::getenv("ODEGPU_STREAM_CHUNK")) s = std::max<Index>(1, std::atoll(e));
    unsigned k = 5;
    while ((Index(1) << k) < s || (N + (Index(1) << k) - 1) >> k > StreamState::kMaxGranules) ++k;
    return k;
}

/// Granule groups moved by one copy each: small first (H2D: the kernel's
/// lanes start on the first granule within tens of microseconds), doubling
/// up to kMaxGroup granules (copies of several MB run at full PCIe rate),
/// and for the copy-out the mirror image — small last, so the D2H left
/// after the kernel's final systems is one granule or two.
std::vector<std::pair<Index, Index>> granule_groups(Index ng, bool small_last) {
    // ODEGPU_STREAM_GROUP_IN / _OUT override the cap (tuning)
    const char* env = std::getenv(small_last ? "ODEGPU_STREAM_GROUP_OUT" : "ODEGPU_STREAM_GROUP_IN");
    const Index kMaxGroup = env ? std::max<Index>(1, std::atoll(env)) : 16;
    std::vector<Index> sizes;
    for (Index g = 0, sz = 1; g < ng; g += sizes.back(), sz = std::min<Index>(2 * sz, kMaxGroup))
        sizes.push_back(std::min(sz, ng - g));
    if (small_last) std::reverse(sizes.begin(), sizes.end());
    std::vector<std::pair<Index, Index>> out;
    Index g = 0;
    for (Index z : sizes) {
        out.emplace_back(g, g + z);
        g += z;
    }
    return out;
}

/// The streaming mode (odegpu_pipeline_mode STREAMING): the whole pool
/// becomes resident in one batch while one persistent solve kernel runs.
/// The pool is cut into granules of 2^shift systems:
///   compute stream: reset gate / flags / outcomes -> [prologue event] ->
///                   solve kernel (a lane takes up a system once its
///                   granule has landed, counts it done when finished)
///   copy-in:        [prologue] -> H2D of a granule group -> gate[0] = its
///                   end (cuStreamWriteValue32), group after group
///   copy-out:       [prologue] -> for a granule group: wait gate[1 + g] >=
///                   granule size for each g (cuStreamWaitValue32) -> D2H
/// The kernel takes the general trig path: the trig certificate needs every
/// system before the launch, and a second launch for systems a certified
/// pass left out would be queued after the copy-out stream's value waits
/// that depend on it — under false serialization of streams (shared
/// hardware queues; compute-sanitizer serialises them outright) a deadlock.
/// A first pass whose input never lands gives up after kStreamTimeoutNs and
/// counts every system done, so no wait is left hanging.
void run_streaming(odegpu_pipeline* p, const Run& j) {
    const odegpu_pool_dims& pd = j.pool->dims;
    const odegpu_system_dims& sd = p->sd;
    const Index N = pd.problem_size;
    const StreamMemOps& ops = stream_memops();
    DeviceGuard g(p->device);
    stream_reserve(p, N);
    StreamState& st = p->stream;
    odegpu_batch* b = st.batch;
    const Index cap = st.cap;
    const odegpu_batch_dims bd{cap, sd.system_dim, sd.param_count, sd.event_count, sd.accessory_count};
    const dev::Controls c = prepare_solve(bd, &p->model, j.cfg, j.ode, j.ev);
    const unsigned shift = stream_granule_shift(N);
    const Index G = Index(1) << shift, NG = (N + G - 1) / G;
    const auto in_groups = granule_groups(NG, false), out_groups = granule_groups(NG, true);
    const odegpu_pool_out none{};
    const odegpu_pool_out& o = j.out ? *j.out : none;
    const bool td_back = o.time_domain && !(o.time_domain == j.pool->time_domain && keeps_time_domain(p->model));
    cudaStream_t cs = b->stream, ci = p->copy_in, co = p->copy_out;
    auto dev_ptr = [](const void* q) { return reinterpret_cast<CUdeviceptr>(q); };
    bool launched = false;
    // ODEGPU_PIPELINE_TRACE=1: per-group H2D / D2H completion times on stderr
    static const bool trace = std::getenv("ODEGPU_PIPELINE_TRACE") != nullptr;
    std::vector<cudaEvent_t> t_in, t_out;
    cudaEvent_t t_zero = nullptr;
    auto mark = [&](std::vector<cudaEvent_t>* v, cudaStream_t s_) {
        if (!trace) return;
        cudaEvent_t e;
        CK(cudaEventCreate(&e));
        CK(cudaEventRecord(e, s_));
        if (v) v->push_back(e);
        else t_zero = e;
    };
    try {
        // prologue on the compute stream
        CK(cudaMemsetAsync(st.gate, 0, sizeof(unsigned) * size_t(1 + NG), cs));
        for (size_t k = 0; k < out_groups.size(); ++k)
            for (Index gi = out_groups[k].first; gi < out_groups[k].second; ++gi)
                st.h_group_of[gi] = static_cast<unsigned short>(k);
        CK(cudaMemcpyAsync(st.group_of, st.h_group_of, sizeof(unsigned short) * size_t(NG), cudaMemcpyHostToDevice,
                           cs));
        CK(cudaMemsetAsync(st.bad, 0, 4 * sizeof(unsigned long long), cs));
        CK(cudaMemsetAsync(st.bad, 0xff, sizeof(unsigned long long), cs)); // no t1 < t0 yet
        CK(cudaMemsetAsync(b->first_bad, 0xff, sizeof(unsigned long long), cs)); // flags[0]: checked in the kernel
        CK(cudaMemsetAsync(b->first_bad + 1, 0xff, sizeof(unsigned long long), cs)); // flags[1]: general trig
        b->a.count = N;
        b->order_count = -1;
        launch_reset_outcomes(b, 0, N);
        CK(cudaEventRecord(st.prologue, cs));
        mark(nullptr, cs);
        CK(cudaStreamWaitEvent(ci, st.prologue, 0));
        CK(cudaStreamWaitEvent(co, st.prologue, 0));

        auto h2d = [&](const std::pair<Index, Index>& grp) {
            const Index s0 = grp.first * G, n = std::min(grp.second * G, N) - s0;
            auto put = [&](Real* dst, const double* src, Index comps) {
                if (!comps) return;
                CK(cudaMemcpy2DAsync(dst + s0, size_t(cap) * 8, src + s0, size_t(N) * 8, size_t(n) * 8, size_t(comps),
                                     cudaMemcpyHostToDevice, ci));
            };
            put(b->a.td, j.pool->time_domain, 2);
            put(b->a.state, j.pool->state, sd.system_dim);
            put(const_cast<Real*>(b->a.params), j.pool->parameters, sd.param_count);
            put(b->a.acc, j.pool->accessories, sd.accessory_count);
            check_cu(ops.write(reinterpret_cast<CUstream>(ci), dev_ptr(st.gate), cuuint32_t(grp.second), 0),
                     "cuStreamWriteValue32");
            mark(&t_in, ci);
        };
        // ODEGPU_STREAM_PRELOAD=1 (diagnostic): the whole pool lands before
        // the kernel starts, which isolates the streaming kernel's own speed
        static const bool preload = std::getenv("ODEGPU_STREAM_PRELOAD") != nullptr;
        // Every H2D group is enqueued BEFORE the kernel, so the kernel only
        // ever waits on work queued ahead of it: were the copy-in and compute
        // streams falsely serialised (shared hardware queue), the copies
        // would simply finish first (less overlap, no deadlock). Enqueueing
        // the ~20 groups takes the host well under a millisecond, while
        // group 0's copy is already running.
        for (const auto& grp : in_groups) h2d(grp);
        if (preload) {
            cudaEvent_t all_in = nullptr;
            CK(cudaEventCreateWithFlags(&all_in, cudaEventDisableTiming));
            CK(cudaEventRecord(all_in, ci));
            CK(cudaStreamWaitEvent(cs, all_in, 0));
            CK(cudaEventDestroy(all_in));
        }
        // the solve kernel over the whole pool, gated per granule
        b->a.gate.ready = st.gate;
        b->a.gate.done = st.gate + 1;
        b->a.gate.group_of = st.group_of;
        b->a.gate.bad = st.bad;
        b->a.gate.packed = o.outcomes ? st.packed : nullptr;
        b->a.gate.shift = shift;
        b->stream_mode = 1;
        b->build_order = false;
        b->fuse_request = j.iterations;
        launch_model(b, p->model, j.cfg->algorithm, c);
        launched = true;
        if (b->fused_done != j.iterations) throw Error(ODEGPU_ERR_CUDA, "streaming: iterations did not fuse");
        // copy-out: each group once all its systems are counted done
        for (size_t k = 0; k < out_groups.size(); ++k) {
            const auto& grp = out_groups[k];
            const Index s0 = grp.first * G, n = std::min(grp.second * G, N) - s0;
            check_cu(ops.wait(reinterpret_cast<CUstream>(co), dev_ptr(st.gate + 1 + k), cuuint32_t(n),
                              CU_STREAM_WAIT_VALUE_GEQ),
                     "cuStreamWaitValue32");
            auto get = [&](double* dst, const Real* src, Index comps) {
                if (!dst || !comps) return;
                CK(cudaMemcpy2DAsync(dst + s0, size_t(N) * 8, src + s0, size_t(cap) * 8, size_t(n) * 8, size_t(comps),
                                     cudaMemcpyDeviceToHost, co));
            };
            if (td_back) get(o.time_domain, b->a.td, 2);
            get(o.state, b->a.state, sd.system_dim);
            get(o.accessories, b->a.acc, sd.accessory_count);
            if (o.outcomes)
                CK(cudaMemcpyAsync(o.outcomes + s0, st.packed + 56 * size_t(s0), 56 * size_t(n),
                                   cudaMemcpyDeviceToHost, co));
            mark(&t_out, co);
        }
        CK(cudaMemcpyAsync(st.h_bad, st.bad, 4 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, cs));
        CK(cudaStreamSynchronize(cs));
        CK(cudaStreamSynchronize(ci));
        CK(cudaStreamSynchronize(co));
        if (trace) {
            float ks = 0, ke = 0;
            cudaEventElapsedTime(&ks, t_zero, b->ev_start);
            cudaEventElapsedTime(&ke, t_zero, b->ev_stop);
            std::fprintf(stderr, "[stream] %lld granules of %lld: kernel %.3f -> %.3f ms\n",
                         static_cast<long long>(NG), static_cast<long long>(G), ks, ke);
            for (size_t k = 0; k < t_in.size() && k < in_groups.size(); ++k) {
                float a = 0;
                cudaEventElapsedTime(&a, t_zero, t_in[k]);
                std::fprintf(stderr, "[stream] in  granules [%lld, %lld): landed %.3f ms\n",
                             static_cast<long long>(in_groups[k].first), static_cast<long long>(in_groups[k].second), a);
            }
            for (size_t k = 0; k < t_out.size(); ++k) {
                float d = 0;
                cudaEventElapsedTime(&d, t_zero, t_out[k]);
                std::fprintf(stderr, "[stream] out granules [%lld, %lld): shipped %.3f ms\n",
                             static_cast<long long>(out_groups[k].first), static_cast<long long>(out_groups[k].second),
                             d);
            }
            for (auto e : t_in) cudaEventDestroy(e);
            for (auto e : t_out) cudaEventDestroy(e);
            cudaEventDestroy(t_zero);
        }
    } catch (...) {
        // release a kernel still waiting on chunks that will not come, then
        // quiesce all three streams before the error returns
        if (launched) {
            cudaStream_t aux = nullptr;
            if (cudaStreamCreateWithFlags(&aux, cudaStreamNonBlocking) == cudaSuccess) {
                ops.write(reinterpret_cast<CUstream>(aux), dev_ptr(st.gate), kStreamAbortHost, 0);
                cudaStreamSynchronize(aux);
                cudaStreamDestroy(aux);
            }
        }
        cudaStreamSynchronize(cs);
        cudaStreamSynchronize(ci);
        cudaStreamSynchronize(co);
        b->stream_mode = 0;
        b->a.gate = dev::StreamGate{};
        b->a.count = cap;
        throw;
    }
    b->stream_mode = 0;
    b->a.gate = dev::StreamGate{};
    b->a.count = cap;
    if (st.h_bad[2]) throw Error(ODEGPU_ERR_CUDA, "streaming: timed out waiting for pool chunks");
    // the index the chunked run reports: the lowest offender's index in its
    // batch_capacity chunk (the reference's run_chunks solves chunk by chunk)
    if (st.h_bad[0] != ~0ull)
        throw_invalid("solve: system " + std::to_string(static_cast<long long>(Index(st.h_bad[0]) % p->cap)) +
                      " has t1 < t0");
}

void run_range(odegpu_pipeline* p, const Run& j, Index begin, Index end) {
    // AUTO runs the chunked slots: measured on one B200 (e2e, bench.py's
    // chunking; profiles/r02v/ vs r02e/, scripts/stream_trace.py) streaming
    // is even with them on cfg4 (36.2 vs 36.8 G steps/s), behind on cfg1
    // (0.78 vs 0.62 ms; all 46 080 lanes finish together, so its D2H cannot
    // overlap) and on cfg2 (3.6 vs 3.2 ms: both modes are PCIe-bound at ~60
    // GB/s both ways, and the slots' copies are larger), and for Keller-
    // Miksis its instantiation runs ~6 % slower. It wins only where chunks
    // are far too small to fill the device (cfg1 in 8 chunks: 0.67 vs 1.05 ms).
    if (begin == 0 && end == j.pool->dims.problem_size && p->mode == ODEGPU_PIPELINE_STREAMING) {
        const char* why = stream_blocker(p, j);
        if (!why) {
            p->last_mode = ODEGPU_PIPELINE_STREAMING;
            run_streaming(p, j);
            return;
        }
        throw_unsupported(std::string("streaming pipeline: ") + why);
    }
    p->last_mode = ODEGPU_PIPELINE_CHUNKED;
    ChunkSource src;
    src.next = begin;
    src.end = end;
    src.step = p->cap;
    run_chunks(p, j, src);
}

void validate_run(const odegpu_pool_view* pool, const odegpu_solver_config* cfg, const odegpu_ode_controls* ode,
                  Index iterations, Index record_from) {
    if (!pool || !cfg || !ode) throw_invalid("solve_pool: null argument");
    if (iterations < 1) throw_invalid("solve_iteratively: iterations must be >= 1");
    if (record_from < 0 || record_from > iterations) throw_invalid("solve_pool: record_from outside [0, iterations]");
    if (pool->dims.problem_size < 1) throw_invalid("PoolDims: problem_size must be >= 1");
    if (!pool->time_domain || !pool->state) throw_invalid("solve_pool: pool arrays missing");
}

} // namespace
} // namespace odegpu::detail

extern "C" {

int odegpu_host_register(void* ptr, size_t bytes) {
    return guarded([&] {
        if (!ptr || bytes == 0) throw_invalid("host_register: empty range");
        CK(cudaHostRegister(ptr, bytes, cudaHostRegisterPortable));
    });
}

int odegpu_host_unregister(void* ptr) {
    return guarded([&] { CK(cudaHostUnregister(ptr)); });
}

int odegpu_slice(odegpu_index total, int parts, int index, odegpu_index* begin, odegpu_index* end) {
    return guarded([&] {
        if (total < 0 || parts < 1 || index < 0 || index >= parts || !begin || !end)
            throw_invalid("slice: bad arguments");
        const Index base = total / parts, extra = total % parts;
        *begin = index * base + std::min<Index>(index, extra);
        *end = *begin + base + (index < extra ? 1 : 0);
    });
}

int odegpu_pipeline_create(const odegpu_model* model, odegpu_index batch_capacity, int device,
                           odegpu_pipeline** out) {
    return guarded([&] {
        if (!model || !out) throw_invalid("null argument");
        *out = nullptr;
        *out = pipeline_create(*model, batch_capacity, device);
    });
}

int odegpu_pipeline_set_mode(odegpu_pipeline* p, int32_t mode) {
    return guarded([&] {
        if (!p) throw_invalid("null pipeline");
        if (mode != ODEGPU_PIPELINE_AUTO && mode != ODEGPU_PIPELINE_CHUNKED && mode != ODEGPU_PIPELINE_STREAMING)
            throw_invalid("pipeline: unknown mode " + std::to_string(mode));
        p->mode = mode;
    });
}

int odegpu_pipeline_last_mode(const odegpu_pipeline* p, int32_t* mode) {
    return guarded([&] {
        if (!p || !mode) throw_invalid("null argument");
        *mode = p->last_mode;
    });
}

void odegpu_pipeline_destroy(odegpu_pipeline* p) {
    if (!p) return;
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(p->device);
    delete p;
    if (prev >= 0) cudaSetDevice(prev);
}

int odegpu_pipeline_run(odegpu_pipeline* p, const odegpu_pool_view* pool, const odegpu_pool_out* out,
                        const odegpu_solver_config* cfg, const odegpu_ode_controls* ode,
                        const odegpu_event_controls* ev, odegpu_index iterations, odegpu_index record_from,
                        uint32_t record_mask, odegpu_chunk_sink on_chunk, void* user) {
    return guarded([&] {
        if (!p) throw_invalid("null pipeline");
        validate_run(pool, cfg, ode, iterations, record_from);
        std::mutex mu;
        const Run j{pool, out, cfg, ode, ev, iterations, record_from, record_mask, on_chunk, user, &mu};
        run_range(p, j, 0, pool->dims.problem_size);
    });
}

int odegpu_pipeline_run_tallied(odegpu_pipeline* p, const odegpu_pool_view* pool, const odegpu_pool_out* out,
                                const odegpu_solver_config* cfg, const odegpu_ode_controls* ode,
                                const odegpu_event_controls* ev, odegpu_index iterations, odegpu_index record_from,
                                uint32_t record_mask, odegpu_chunk_sink on_chunk, void* user,
                                odegpu_scan_tally* tally) {
    return guarded([&] {
        if (!p || !tally) throw_invalid("null argument");
        validate_run(pool, cfg, ode, iterations, record_from);
        std::mutex mu;
        Run j{pool, out, cfg, ode, ev, iterations, record_from, record_mask, on_chunk, user, &mu};
        j.tally = tally;
        run_range(p, j, 0, pool->dims.problem_size);
    });
}

int odegpu_solve_pool(const odegpu_pool_view* pool, const odegpu_pool_out* out, const odegpu_model* model,
                      const odegpu_solver_config* cfg, const odegpu_ode_controls* ode,
                      const odegpu_event_controls* ev, odegpu_index batch_capacity, odegpu_index iterations,
                      odegpu_index record_from, uint32_t record_mask, odegpu_chunk_sink on_chunk, void* user,
                      int device) {
    return guarded([&] {
        if (!model) throw_invalid("solve_pool: null argument");
        validate_run(pool, cfg, ode, iterations, record_from);
        const Index cap = batch_capacity < 1 ? batch_capacity : std::min<Index>(batch_capacity, pool->dims.problem_size);
        odegpu_pipeline* p = pipeline_create(*model, cap, device);
        std::mutex mu;
        const Run j{pool, out, cfg, ode, ev, iterations, record_from, record_mask, on_chunk, user, &mu};
        try {
            run_range(p, j, 0, pool->dims.problem_size);
        } catch (...) {
            delete p;
            throw;
        }
        delete p;
    });
}

int odegpu_solve_pool_multi(const odegpu_pool_view* pool, const odegpu_pool_out* out, const odegpu_model* model,
                            const odegpu_solver_config* cfg, const odegpu_ode_controls* ode,
                            const odegpu_event_controls* ev, odegpu_index batch_capacity,
                            odegpu_index iterations, odegpu_index record_from, uint32_t record_mask,
                            odegpu_chunk_sink on_chunk, void* user, const int* devices, int n_devices) {
    return odegpu_solve_pool_multi_tallied(pool, out, model, cfg, ode, ev, batch_capacity, iterations, record_from,
                                           record_mask, on_chunk, user, devices, n_devices, 0, nullptr);
}

int odegpu_solve_pool_multi_tallied(const odegpu_pool_view* pool, const odegpu_pool_out* out,
                                    const odegpu_model* model, const odegpu_solver_config* cfg,
                                    const odegpu_ode_controls* ode, const odegpu_event_controls* ev,
                                    odegpu_index batch_capacity, odegpu_index iterations, odegpu_index record_from,
                                    uint32_t record_mask, odegpu_chunk_sink on_chunk, void* user,
                                    const int* devices, int n_devices, int chunk_aligned, odegpu_scan_tally* tally) {
    return guarded([&] {
        if (!devices || n_devices < 1) throw_invalid("solve_pool_multi: no devices");
        if (!model) throw_invalid("solve_pool: null argument");
        validate_run(pool, cfg, ode, iterations, record_from);
        if (batch_capacity < 1) throw_invalid("BatchDims: batch_capacity must be >= 1");
        std::mutex mu;
        Run j{pool, out, cfg, ode, ev, iterations, record_from, record_mask, on_chunk, user, &mu};
        j.tally = tally;
        std::exception_ptr* failures = new std::exception_ptr[size_t(n_devices)];
        std::vector<std::thread> threads;
        const Index N = pool->dims.problem_size;
        // one queue of chunks of batch_capacity systems in pool order, shared
        // by all devices; chunk boundaries do not depend on the device count,
        // so per-chunk results (and scan rows) equal the single-device run's
        std::atomic<Index> queue{0};
        const Index cap = std::min<Index>(batch_capacity, N);
        (void)chunk_aligned; // chunks are always aligned to batch_capacity now
        for (int d = 0; d < n_devices; ++d) {
            const Run* jp = &j;
            std::exception_ptr* slot = failures + d;
            const int dev_id = devices[d];
            const odegpu_model m = *model;
            std::atomic<Index>* q = &queue;
            threads.emplace_back([jp, slot, dev_id, m, cap, q, N] {
                odegpu_pipeline* p = nullptr;
                try {
                    p = pipeline_create(m, cap, dev_id);
                    ChunkSource src;
                    src.shared = q;
                    src.end = N;
                    src.step = cap;
                    run_chunks(p, *jp, src);
                } catch (...) {
                    *slot = std::current_exception();
                    q->store(N); // the other devices stop claiming chunks
                }
                delete p;
            });
        }
        for (auto& t : threads) t.join();
        std::exception_ptr first;
        for (int d = 0; d < n_devices && !first; ++d) first = failures[d];
        delete[] failures;
        if (first) std::rethrow_exception(first); // first device's error wins (solve.hpp:127 analogue)
    });
}

} // extern "C"
