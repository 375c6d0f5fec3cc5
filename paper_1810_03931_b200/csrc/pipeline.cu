// pipeline.cu — chunked problem-pool batching (the device side of
// src/scan.cpp:88-112 run_chunks) with double-buffered H2D/D2H on two
// streams, and its multi-GPU form (one host thread and one contiguous slice
// per device; no inter-GPU traffic: systems are independent).
#include <cuda_runtime.h>

#include <cstring>
#include <exception>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "internal.cuh"

using namespace odegpu;
using namespace odegpu::detail;

namespace odegpu::detail {

void OutcomeStage::allocate(Index cap) {
    const size_t n = size_t(cap);
    const size_t bytes = n * (8 * 6 + 1) + 64;
    CK(cudaMallocHost(&block, bytes));
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
    if (block) cudaFreeHost(block);
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

/// Host staging of one pipeline slot (pinned).
struct Slot {
    odegpu_batch* batch = nullptr;
    cudaEvent_t done = nullptr;
    double* rec_td = nullptr;   // [n_rec][2][cap]
    double* rec_y = nullptr;    // [n_rec][dim][cap]
    double* rec_acc = nullptr;  // [n_rec][acc][cap]
    std::vector<OutcomeStage> rec_out;
    double* fin_td = nullptr;   // [2][cap]
    double* fin_y = nullptr;
    double* fin_acc = nullptr;
    OutcomeStage fin_out;
    Index start = 0, count = 0;
    bool busy = false;
};

struct PoolJob {
    const odegpu_pool_view* pool;
    const odegpu_pool_out* out;
    const odegpu_model* model;
    const odegpu_solver_config* cfg;
    const odegpu_ode_controls* ode;
    const odegpu_event_controls* ev;
    Index capacity, iterations, record_from;
    uint32_t mask;
    odegpu_chunk_sink sink;
    void* user;
    std::mutex* sink_mutex; // serialises sinks across device threads
};

/// Runs systems [begin, end) of the pool on `device`.
void run_range(const PoolJob& j, Index begin, Index end, int device) {
    const odegpu_pool_dims& pd = j.pool->dims;
    const odegpu_system_dims sd = dims_of(*j.model);
    if (sd.system_dim != pd.system_dim || sd.param_count != pd.param_count ||
        sd.accessory_count != pd.accessory_count)
        throw_invalid("solve_pool: definition and pool dimensions disagree");
    const Index total = end - begin;
    if (total <= 0) return;
    const Index cap = std::min(j.capacity, total);
    const odegpu_batch_dims bd{cap, sd.system_dim, sd.param_count, sd.event_count, sd.accessory_count};
    const dev::Controls c = prepare_solve(bd, j.model, j.cfg, j.ode, j.ev);
    const Index n_rec = j.iterations - j.record_from;
    const Index N = pd.problem_size;
    const bool r_td = j.mask & 1u, r_y = j.mask & 2u, r_acc = (j.mask & 8u) && sd.accessory_count,
               r_out = j.mask & 16u;

    DeviceGuard g(device);
    Slot slots[2];
    auto cleanup = [&] {
        for (auto& s : slots) {
            if (s.batch) odegpu_batch_destroy(s.batch);
            if (s.done) cudaEventDestroy(s.done);
            for (double* p : {s.rec_td, s.rec_y, s.rec_acc, s.fin_td, s.fin_y, s.fin_acc})
                if (p) cudaFreeHost(p);
            for (auto& o : s.rec_out) o.release();
            s.fin_out.release();
        }
    };
    try {
        for (auto& s : slots) {
            s.batch = batch_create(bd, device);
            CK(cudaEventCreateWithFlags(&s.done, cudaEventDisableTiming));
            auto pin = [&](double** p, Index doubles) {
                if (doubles > 0) CK(cudaMallocHost(p, size_t(doubles) * 8));
            };
            if (r_td) pin(&s.rec_td, n_rec * 2 * cap);
            if (r_y) pin(&s.rec_y, n_rec * sd.system_dim * cap);
            if (r_acc) pin(&s.rec_acc, n_rec * sd.accessory_count * cap);
            if (r_out) {
                s.rec_out.resize(size_t(n_rec));
                for (auto& o : s.rec_out) o.allocate(cap);
            }
            if (j.out && j.out->time_domain) pin(&s.fin_td, 2 * cap);
            if (j.out && j.out->state) pin(&s.fin_y, sd.system_dim * cap);
            if (j.out && j.out->accessories && sd.accessory_count) pin(&s.fin_acc, sd.accessory_count * cap);
            if (j.out && j.out->outcomes) s.fin_out.allocate(cap);
        }

        std::vector<odegpu_outcome> packed(size_t(cap) * size_t(std::max<Index>(n_rec, 1)));
        // Consume a finished slot: validation flag, write-back, sink.
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
            if (s.fin_td) put(j.out->time_domain, s.fin_td, 2);
            if (s.fin_y) put(j.out->state, s.fin_y, sd.system_dim);
            if (s.fin_acc) put(j.out->accessories, s.fin_acc, sd.accessory_count);
            if (s.fin_out.block) s.fin_out.pack(j.out->outcomes + off, n);
            if (j.sink && n_rec > 0) {
                if (r_out)
                    for (Index r = 0; r < n_rec; ++r) s.rec_out[size_t(r)].pack(packed.data() + r * n, n);
                // compact the recorded arrays from stride cap to stride n
                auto compact = [&](double* p, Index comps) {
                    if (!p || n == cap) return;
                    for (Index r = 0; r < n_rec; ++r)
                        for (Index cc = 0; cc < comps; ++cc)
                            std::memmove(p + (r * comps + cc) * n, p + (r * comps + cc) * cap, size_t(n) * 8);
                };
                compact(s.rec_td, 2);
                compact(s.rec_y, sd.system_dim);
                compact(s.rec_acc, sd.accessory_count);
                const odegpu_chunk_record rec{s.rec_td, s.rec_y, s.rec_acc, r_out ? packed.data() : nullptr};
                int rc;
                {
                    std::lock_guard<std::mutex> lock(*j.sink_mutex);
                    rc = j.sink(off, n, n_rec, &rec, j.user);
                }
                if (rc != 0) throw Error(rc, "solve_pool: chunk sink returned " + std::to_string(rc));
            }
        };

        int k = 0;
        for (Index start = begin; start < end; start += cap, ++k) {
            Slot& s = slots[k & 1];
            drain(s); // the slot's previous chunk must be consumed before reuse
            odegpu_batch* b = s.batch;
            const Index n = std::min(cap, end - start);
            s.start = start;
            s.count = n;
            b->a.count = n;
            // linear_set(All) of the chunk: pool -> batch, fresh outcomes (batch.cpp:78-104)
            copy_h2d_strided(b->a.td, cap, 0, j.pool->time_domain, N, start, n, 2, b->stream);
            copy_h2d_strided(b->a.state, cap, 0, j.pool->state, N, start, n, sd.system_dim, b->stream);
            if (sd.param_count)
                copy_h2d_strided(const_cast<Real*>(b->a.params), cap, 0, j.pool->parameters, N, start, n,
                                 sd.param_count, b->stream);
            if (sd.accessory_count)
                copy_h2d_strided(b->a.acc, cap, 0, j.pool->accessories, N, start, n, sd.accessory_count, b->stream);
            launch_reset_outcomes(b, 0, n);
            for (Index it = 0; it < j.iterations; ++it) {
                enqueue_time_check(b);
                launch_model(b, *j.model, j.cfg->algorithm, c);
                if (it >= j.record_from) {
                    const Index r = it - j.record_from;
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
            if (s.fin_td) copy_d2h_strided(s.fin_td, cap, 0, b->a.td, cap, 0, n, 2, b->stream);
            if (s.fin_y) copy_d2h_strided(s.fin_y, cap, 0, b->a.state, cap, 0, n, sd.system_dim, b->stream);
            if (s.fin_acc)
                copy_d2h_strided(s.fin_acc, cap, 0, b->a.acc, cap, 0, n, sd.accessory_count, b->stream);
            if (s.fin_out.block) s.fin_out.fetch(b, 0, n, b->stream);
            CK(cudaMemcpyAsync(b->host_flag, b->first_bad, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                               b->stream));
            CK(cudaEventRecord(s.done, b->stream));
            s.busy = true;
            // chunk k-1 (other slot) is drained at the top of iteration k+1, so
            // its D2H and the host work overlap chunk k's kernels
        }
        drain(slots[k & 1]); // oldest first
        drain(slots[(k + 1) & 1]);
    } catch (...) {
        for (auto& s : slots)
            if (s.batch) cudaStreamSynchronize(s.batch->stream);
        cleanup();
        throw;
    }
    cleanup();
}

void validate_job(const PoolJob& j) {
    if (!j.pool || !j.model || !j.cfg || !j.ode) throw_invalid("solve_pool: null argument");
    if (j.capacity < 1) throw_invalid("BatchDims: batch_capacity must be >= 1");
    if (j.iterations < 1) throw_invalid("solve_iteratively: iterations must be >= 1");
    if (j.record_from < 0 || j.record_from > j.iterations)
        throw_invalid("solve_pool: record_from outside [0, iterations]");
    if (j.pool->dims.problem_size < 1) throw_invalid("PoolDims: problem_size must be >= 1");
    if (!j.pool->time_domain || !j.pool->state) throw_invalid("solve_pool: pool arrays missing");
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

int odegpu_solve_pool(const odegpu_pool_view* pool, const odegpu_pool_out* out, const odegpu_model* model,
                      const odegpu_solver_config* cfg, const odegpu_ode_controls* ode,
                      const odegpu_event_controls* ev, odegpu_index batch_capacity, odegpu_index iterations,
                      odegpu_index record_from, uint32_t record_mask, odegpu_chunk_sink on_chunk, void* user,
                      int device) {
    return guarded([&] {
        std::mutex mu;
        const PoolJob j{pool, out, model, cfg, ode, ev, batch_capacity, iterations, record_from, record_mask,
                        on_chunk, user, &mu};
        validate_job(j);
        run_range(j, 0, pool->dims.problem_size, device);
    });
}

int odegpu_solve_pool_multi(const odegpu_pool_view* pool, const odegpu_pool_out* out, const odegpu_model* model,
                            const odegpu_solver_config* cfg, const odegpu_ode_controls* ode,
                            const odegpu_event_controls* ev, odegpu_index batch_capacity,
                            odegpu_index iterations, odegpu_index record_from, uint32_t record_mask,
                            odegpu_chunk_sink on_chunk, void* user, const int* devices, int n_devices) {
    return guarded([&] {
        if (!devices || n_devices < 1) throw_invalid("solve_pool_multi: no devices");
        std::mutex mu;
        const PoolJob j{pool, out, model, cfg, ode, ev, batch_capacity, iterations, record_from, record_mask,
                        on_chunk, user, &mu};
        validate_job(j);
        std::exception_ptr* failures = new std::exception_ptr[size_t(n_devices)];
        std::vector<std::thread> threads;
        for (int d = 0; d < n_devices; ++d) {
            Index b0 = 0, b1 = 0;
            odegpu_slice(pool->dims.problem_size, n_devices, d, &b0, &b1);
            const PoolJob* jp = &j;
            std::exception_ptr* slot = failures + d;
            const int dev_id = devices[d];
            threads.emplace_back([jp, slot, dev_id, b0, b1] {
                try {
                    run_range(*jp, b0, b1, dev_id);
                } catch (...) {
                    *slot = std::current_exception();
                }
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
