// batch.hpp — SolverBatch of the C++ host API: a device-resident SoA batch
// (libodegpu, include/odegpu.h) with a lazily synchronised host mirror, so
// code written against the reference's span accessors
// (/root/reference/proj/include/odensemble/batch.hpp:17-67) keeps working.
//
// Coherence protocol per array (time domain, state, parameters,
// accessories, outcomes):
//   * const accessors copy device -> host only if the mirror is stale; the
//     span they return is a snapshot, valid until the next device operation
//     (re-acquire it afterwards);
//   * non-const accessors hand out a span into live storage, as the
//     reference's do (batch.hpp:24-34): from then on the array is LIVE — it is
//     uploaded before every device operation and downloaded right after every
//     device operation that modifies it, so writes through a span taken before
//     a solve() reach the device and the span shows the solve's results, as
//     with the reference's host vectors. detach_spans() ends that (outstanding
//     mutable spans must then be re-acquired) and returns to lazy transfers;
//   * device operations (linear_set, random_set, solve) invalidate the
//     mirror of what they modify.
// Transient iterations therefore cost no PCIe traffic unless a sink reads or
// a mutable span is outstanding.
#ifndef ODEGPU_BATCH_HPP
#define ODEGPU_BATCH_HPP

#include <limits>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "odegpu.h"
#include "odegpu/core.hpp"
#include "odegpu/pool.hpp"

namespace odegpu {

/// driver.hpp:34-42 — byte-compatible with odegpu_outcome.
struct SystemOutcome {
    Real final_t = 0;
    StopReason reason = StopReason::ReachedEndTime;
    Index accepted_steps = 0;
    Index rejected_steps = 0;
    Index event_detections = 0;
    Index secant_failures = 0;
    Real smallest_step = std::numeric_limits<Real>::infinity();
};
static_assert(sizeof(SystemOutcome) == sizeof(odegpu_outcome), "SystemOutcome layout");

/// driver.hpp:25-30 (tile_size / worker_count validated, scheduling is the GPU's).
struct SolverConfig {
    Algorithm algorithm = Algorithm::RKCK45;
    Real initial_time_step = 1e-3;
    Index tile_size = 64;
    Index worker_count = 1;
};

namespace detail {

/// Rethrows a C-ABI failure with the reference's exception class.
[[noreturn]] inline void rethrow(int rc) {
    const std::string msg = odegpu_last_error();
    if (rc == ODEGPU_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
    if (rc == ODEGPU_ERR_OUT_OF_RANGE) throw std::out_of_range(msg);
    throw std::runtime_error(msg);
}
inline void check(int rc) {
    if (rc != ODEGPU_OK) rethrow(rc);
}

} // namespace detail

class SolverBatch {
public:
    explicit SolverBatch(const BatchDims& dims, int device = 0) : dims_(dims) {
        dims.validate();
        const odegpu_batch_dims d{dims.batch_capacity, dims.system_dim, dims.param_count, dims.event_count,
                                  dims.accessory_count};
        detail::check(odegpu_batch_create(&d, device, &h_));
        const auto n = static_cast<std::size_t>(dims.batch_capacity);
        host_[kTd].assign(2 * n, 0.0);
        host_[kState].assign(static_cast<std::size_t>(dims.system_dim) * n, 0.0);
        host_[kParams].assign(static_cast<std::size_t>(dims.param_count) * n, 0.0);
        host_[kAcc].assign(static_cast<std::size_t>(dims.accessory_count) * n, 0.0);
        outcomes_.assign(n, SystemOutcome{});
    }
    SolverBatch(const SolverBatch&) = delete;
    SolverBatch& operator=(const SolverBatch&) = delete;
    SolverBatch(SolverBatch&& o) noexcept { swap(o); }
    SolverBatch& operator=(SolverBatch&& o) noexcept {
        swap(o);
        return *this;
    }
    ~SolverBatch() { odegpu_batch_destroy(h_); }

    const BatchDims& dims() const { return dims_; }
    Index size() const { return dims_.batch_capacity; }
    odegpu_batch* handle() const { return h_; }

    std::span<Real> time_domain() { return writable(kTd); }
    std::span<Real> state() { return writable(kState); }
    std::span<Real> parameters() { return writable(kParams); }
    std::span<Real> accessories() { return writable(kAcc); }
    std::span<const Real> time_domain() const { return readable(kTd); }
    std::span<const Real> state() const { return readable(kState); }
    std::span<const Real> parameters() const { return readable(kParams); }
    std::span<const Real> accessories() const { return readable(kAcc); }

    std::span<SystemOutcome> outcomes() {
        pull_outcomes();
        dirty_[kOut] = true;
        live_[kOut] = true;
        return outcomes_;
    }
    std::span<const SystemOutcome> outcomes() const {
        pull_outcomes();
        return outcomes_;
    }

    Real time_start(Index i) const { return readable(kTd)[idx(i, 0)]; }
    Real time_end(Index i) const { return readable(kTd)[idx(i, 1)]; }
    Real state_at(Index i, Index c) const { return readable(kState)[idx(i, c)]; }
    Real param_at(Index i, Index c) const { return readable(kParams)[idx(i, c)]; }
    Real accessory_at(Index i, Index c) const { return readable(kAcc)[idx(i, c)]; }

    /// Order in which the solve kernel takes up systems (ODEGPU_FETCH_*,
    /// odegpu_batch_set_fetch_order); never changes a result.
    void set_fetch_order(int mode) { detail::check(odegpu_batch_set_fetch_order(h_, mode)); }

    /// batch.cpp:42-44
    void reset_outcomes() {
        push();
        detail::check(odegpu_batch_reset_outcomes(h_));
        valid_[kOut] = false;
    }

    /// Upload every array the host modified or may have modified through an
    /// outstanding mutable span (before a device operation).
    void push() {
        for (int k = 0; k < 4; ++k)
            if (dirty_[k] || live_[k]) {
                if (!host_[k].empty()) detail::check(odegpu_batch_write(h_, k, host_[k].data()));
                dirty_[k] = false;
            }
        if (dirty_[kOut] || live_[kOut]) {
            detail::check(odegpu_batch_write_outcomes(h_, reinterpret_cast<const odegpu_outcome*>(outcomes_.data())));
            dirty_[kOut] = false;
        }
    }
    /// The device modified arrays `mask` (bit k = array k, bit 4 = outcomes):
    /// live arrays are refreshed now (their spans must show the new values),
    /// the others on their next access.
    void invalidate_host(unsigned mask) {
        for (int k = 0; k < 5; ++k)
            if (mask & (1u << k)) {
                valid_[k] = false;
                if (live_[k]) {
                    if (k == kOut) pull_outcomes();
                    else readable(k);
                }
            }
    }
    /// Mutable spans handed out so far become invalid (re-acquire them);
    /// transfers go back to lazy (see the coherence protocol above).
    void detach_spans() {
        push();
        for (bool& l : live_) l = false;
    }

private:
    enum { kTd = 0, kState = 1, kParams = 2, kAcc = 3, kOut = 4 };

    std::size_t idx(Index i, Index c) const { return static_cast<std::size_t>(flat_index(i, c, size())); }

    std::span<const Real> readable(int k) const {
        if (!valid_[k]) {
            if (!host_[k].empty()) detail::check(odegpu_batch_read(h_, k, host_[k].data()));
            valid_[k] = true;
        }
        return host_[k];
    }
    std::span<Real> writable(int k) {
        readable(k);
        dirty_[k] = true;
        live_[k] = true;
        return host_[k];
    }
    void pull_outcomes() const {
        if (!valid_[kOut]) {
            detail::check(odegpu_batch_read_outcomes(h_, reinterpret_cast<odegpu_outcome*>(outcomes_.data())));
            valid_[kOut] = true;
        }
    }
    void swap(SolverBatch& o) noexcept {
        std::swap(dims_, o.dims_);
        std::swap(h_, o.h_);
        for (int k = 0; k < 4; ++k) std::swap(host_[k], o.host_[k]);
        std::swap(outcomes_, o.outcomes_);
        for (int k = 0; k < 5; ++k) {
            std::swap(valid_[k], o.valid_[k]);
            std::swap(dirty_[k], o.dirty_[k]);
            std::swap(live_[k], o.live_[k]);
        }
    }

    BatchDims dims_{};
    odegpu_batch* h_ = nullptr;
    mutable std::vector<Real> host_[4];
    mutable std::vector<SystemOutcome> outcomes_;
    mutable bool valid_[5] = {true, true, true, true, true}; // fresh batch: zeros on both sides
    bool dirty_[5] = {false, false, false, false, false};
    bool live_[5] = {false, false, false, false, false}; // a mutable span is outstanding
};

/// batch.cpp:78-104 — pool[start_in_pool, +n) -> batch[start_in_batch, +n).
inline void linear_set(SolverBatch& batch, const ProblemPool& pool, const LinearCopySpec& spec) {
    batch.push();
    const odegpu_pool_view v = pool.view();
    const odegpu_linear_copy_spec s{spec.start_in_batch, spec.start_in_pool, spec.element_count,
                                    static_cast<int32_t>(spec.copy_mode), 0};
    detail::check(odegpu_linear_set(batch.handle(), &v, &s));
    const unsigned props = spec.copy_mode == CopyMode::All ? 0xFu : (1u << static_cast<int>(spec.copy_mode));
    batch.invalidate_host(props | 0x10u);
}

/// batch.cpp:106-135 — batch[ib[j]] = pool[ip[j]].
inline void random_set(SolverBatch& batch, const ProblemPool& pool, const RandomCopySpec& spec) {
    if (spec.indices_in_batch.size() != spec.indices_in_pool.size())
        throw std::invalid_argument("random_set: index lists differ in length");
    batch.push();
    const odegpu_pool_view v = pool.view();
    detail::check(odegpu_random_set(batch.handle(), &v, spec.indices_in_batch.data(), spec.indices_in_pool.data(),
                                    static_cast<odegpu_index>(spec.indices_in_batch.size()),
                                    static_cast<int32_t>(spec.copy_mode)));
    const unsigned props = spec.copy_mode == CopyMode::All ? 0xFu : (1u << static_cast<int>(spec.copy_mode));
    batch.invalidate_host(props | 0x10u);
}

} // namespace odegpu

#endif
