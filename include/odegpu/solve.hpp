// solve.hpp — the drop-in entry points of the C++ host API:
// solve (/root/reference/proj/include/odensemble/solve.hpp:60-128) and
// solve_iteratively (solve.hpp:133-142), running on the GPU through the C ABI.
//
// Validation and its messages are the reference's (performed in libodegpu);
// failures are rethrown as std::invalid_argument / std::out_of_range.
// solve() is synchronous like the reference. Of the host observers
// (SolveObservers, solve.hpp:36-50) the detection observer is supported:
// the device records every detection in a log and on_detection runs on the
// calling thread after the solve, per system in the order the driver made
// them (the reference runs it on worker threads, systems interleaved). A
// per-step observer cannot run on the device: passing one
// is a compile error; per-solve tallies come from SolverBatch diagnostics.
#ifndef ODEGPU_SOLVE_HPP
#define ODEGPU_SOLVE_HPP

#include <cstdint>
#include <exception>
#include <span>
#include <type_traits>
#include <stdexcept>
#include <utility>
#include <vector>

#include "odegpu.h"
#include "odegpu/batch.hpp"
#include "odegpu/system.hpp"

namespace odegpu {

/// How a detection step met the zone (events.hpp:28-31).
enum class DetectionKind : std::uint8_t { SteppedAcross, EnteredFromAbove, EnteredFromBelow };

/// One recorded event detection (events.hpp:36-47).
struct Detection {
    Index event_index = 0;
    DetectionKind kind = DetectionKind::SteppedAcross;
    Real t = 0;
    Real value = 0;
    Index counter = 0;
    bool in_zone = false;
};

/// Observer no-ops and bundle (solve.hpp:36-50).
struct NoBatchStepObserver {
    void operator()(Index, Real, std::span<const Real>) const {}
};
struct NoBatchDetectionObserver {
    void operator()(Index, const Detection&, std::span<const Real>, std::span<const Real>) const {}
};
template <typename StepObs = NoBatchStepObserver, typename DetObs = NoBatchDetectionObserver>
struct SolveObservers {
    StepObs on_step{};
    DetObs on_detection{};
};

namespace detail {

/// Materialised controls (solve.hpp:153-155) with C views into them.
struct CControls {
    OdeControls ode;
    EventControls ev;
    std::vector<int32_t> dir;
    odegpu_ode_controls c_ode{};
    odegpu_event_controls c_ev{};
    odegpu_solver_config c_cfg{};

    template <SystemModel D>
    CControls(const D& def, const SolverConfig& cfg) : ode(def.ode_controls()), ev(def.event_controls()) {
        dir.assign(ev.direction.begin(), ev.direction.end());
        c_ode = {ode.rel_tol.data(), ode.abs_tol.data(), ode.max_step, ode.min_step, ode.step_grow_limit,
                 ode.step_shrink_limit};
        c_ev = {dir.data(), ev.tolerance.data(), ev.stop_condition.data(), ev.max_steps_in_zone};
        c_cfg = {static_cast<int32_t>(cfg.algorithm), 0, cfg.initial_time_step, cfg.tile_size, cfg.worker_count};
        const SystemDims d = def.dims();
        if (static_cast<Index>(ode.rel_tol.size()) != d.system_dim ||
            static_cast<Index>(ode.abs_tol.size()) != d.system_dim)
            throw std::invalid_argument("solve: ode controls length != system_dim");
        if (static_cast<Index>(ev.direction.size()) != d.event_count ||
            static_cast<Index>(ev.tolerance.size()) != d.event_count ||
            static_cast<Index>(ev.stop_condition.size()) != d.event_count)
            throw std::invalid_argument("solve: event controls length != event_count");
    }
};

constexpr unsigned kSolveWrites = 0x1Bu; // time domain, state, accessories, outcomes (params never)

} // namespace detail

/// User-defined models are solved by a kernel instantiated in the caller's
/// nvcc translation unit: include "odegpu/device/custom.cuh" there.
template <SystemModel D>
void solve_custom(SolverBatch& batch, const D& def, const SolverConfig& cfg);

namespace detail {

template <BuiltinModel D>
void solve_builtin(SolverBatch& batch, const D& def, const SolverConfig& cfg) {
    CControls c(def, cfg);
    const odegpu_model m = def.descriptor();
    batch.push();
    const int rc = odegpu_solve(batch.handle(), &m, &c.c_cfg, &c.c_ode, &c.c_ev);
    batch.invalidate_host(kSolveWrites);
    check(rc);
}

/// odegpu_solve_iteratively with a C trampoline around the C++ sink (NULL
/// sink when `sink` is null: iterations back to back on the device).
template <BuiltinModel D, typename Sink>
void solve_iteratively_builtin(SolverBatch& batch, const D& def, const SolverConfig& cfg, Index iterations,
                               Sink* sink) {
    CControls c(def, cfg);
    const odegpu_model m = def.descriptor();
    batch.push();
    struct Ctx {
        SolverBatch* batch;
        Sink* sink;
        std::exception_ptr error;
    } ctx{&batch, sink, nullptr};
    const auto trampoline = [](odegpu_index it, odegpu_batch*, void* user) -> int {
        auto* x = static_cast<Ctx*>(user);
        x->batch->invalidate_host(kSolveWrites);
        try {
            (*x->sink)(static_cast<Index>(it), static_cast<const SolverBatch&>(*x->batch));
            x->batch->push(); // a sink may not write, but keep the mirror coherent regardless
            return 0;
        } catch (...) {
            x->error = std::current_exception();
            return 1;
        }
    };
    const int rc = odegpu_solve_iteratively(batch.handle(), &m, &c.c_cfg, &c.c_ode, &c.c_ev, iterations,
                                            sink ? +trampoline : nullptr, sink ? &ctx : nullptr);
    batch.invalidate_host(kSolveWrites);
    if (ctx.error) std::rethrow_exception(ctx.error);
    check(rc);
}

struct NoSink {
    void operator()(Index, const SolverBatch&) const {}
};

} // namespace detail

namespace detail {

template <typename StepObs, typename DetObs>
constexpr bool kObservesDetections = !std::is_same_v<std::remove_cvref_t<DetObs>, NoBatchDetectionObserver>;

template <typename StepObs>
constexpr void require_no_step_observer() {
    static_assert(std::is_same_v<std::remove_cvref_t<StepObs>, NoBatchStepObserver>,
                  "odegpu: a per-step observer (on_step) cannot run on the device; use SolverBatch diagnostics");
}

/// Runs `solve_one` with the batch's detection log enabled, then hands each
/// record to on_detection in (system, sequence) order. The log starts at 4
/// records per system; a solve that detects more is repeated from a device
/// copy of its inputs with a log large enough (results are deterministic).
template <typename DetObs, typename SolveOne>
void with_detection_log(SolverBatch& batch, DetObs& on_detection, SolveOne&& solve_one) {
    const Index dim = batch.dims().system_dim;
    Index cap = 4 * batch.size();
    odegpu_index count = 0, total = 0;
    batch.push();
    const auto dd = batch.dims();
    const odegpu_batch_dims bd{dd.batch_capacity, dd.system_dim, dd.param_count, dd.event_count, dd.accessory_count};
    odegpu_batch* before = nullptr;
    check(odegpu_batch_create(&bd, odegpu_batch_device(batch.handle()), &before));
    struct Release {
        odegpu_batch* b;
        ~Release() { odegpu_batch_destroy(b); }
    } release{before};
    check(odegpu_batch_copy(before, batch.handle()));
    check(odegpu_batch_set_detection_log(batch.handle(), cap));
    solve_one();
    check(odegpu_batch_read_detection_log(batch.handle(), nullptr, nullptr, nullptr, 0, &count, &total));
    if (total > cap) { // overflowed: the same inputs again, with room for every record
        cap = total;
        check(odegpu_batch_copy(batch.handle(), before));
        check(odegpu_batch_set_detection_log(batch.handle(), cap));
        solve_one();
    }
    std::vector<odegpu_detection> rec(static_cast<std::size_t>(total));
    std::vector<Real> pre(static_cast<std::size_t>(total * dim)), post(static_cast<std::size_t>(total * dim));
    const int rc = odegpu_batch_read_detection_log(batch.handle(), rec.data(), pre.data(), post.data(), total, &count,
                                                   &total);
    check(odegpu_batch_set_detection_log(batch.handle(), 0));
    check(rc);
    for (odegpu_index k = 0; k < count; ++k) {
        const odegpu_detection& r = rec[static_cast<std::size_t>(k)];
        const Detection d{r.event_index, static_cast<DetectionKind>(r.kind), r.t, r.value, r.counter, r.in_zone != 0};
        on_detection(static_cast<Index>(r.system), d,
                     std::span<const Real>(pre.data() + k * dim, static_cast<std::size_t>(dim)),
                     std::span<const Real>(post.data() + k * dim, static_cast<std::size_t>(dim)));
    }
}

} // namespace detail

/// Integrates every system of the batch on the GPU (solve.hpp:60-128).
/// Built-in models run through the C ABI; other SystemModels through a
/// kernel instantiated from include/odegpu/device/custom.cuh.
template <SystemModel D>
void solve(SolverBatch& batch, const D& def, const SolverConfig& cfg = {}) {
    if constexpr (BuiltinModel<D>)
        detail::solve_builtin(batch, def, cfg);
    else
        solve_custom(batch, def, cfg);
}

/// solve() with observers (solve.hpp:60-63): on_detection receives every
/// detection of the solve (see the file comment for the order).
template <SystemModel D, typename StepObs, typename DetObs>
void solve(SolverBatch& batch, const D& def, const SolverConfig& cfg, SolveObservers<StepObs, DetObs> observers) {
    detail::require_no_step_observer<StepObs>();
    if constexpr (!detail::kObservesDetections<StepObs, DetObs> || !BuiltinModel<D>) {
        static_assert(!detail::kObservesDetections<StepObs, DetObs> || BuiltinModel<D>,
                      "odegpu: the detection log is available for the built-in models");
        solve(batch, def, cfg);
    } else {
        detail::with_detection_log(batch, observers.on_detection, [&] { detail::solve_builtin(batch, def, cfg); });
    }
}

/// solve.hpp:133-142: `iterations` solves, sink(i, const batch&) after each.
template <SystemModel D, typename Sink>
void solve_iteratively(SolverBatch& batch, const D& def, const SolverConfig& cfg, Index iterations, Sink&& sink) {
    if (iterations < 1) throw std::invalid_argument("solve_iteratively: iterations must be >= 1");
    if constexpr (BuiltinModel<D>) {
        using S = std::remove_reference_t<Sink>;
        detail::solve_iteratively_builtin<D, S>(batch, def, cfg, iterations, &sink);
    } else {
        for (Index i = 0; i < iterations; ++i) {
            solve_custom(batch, def, cfg);
            sink(i, static_cast<const SolverBatch&>(batch));
        }
    }
}

/// solve_iteratively with observers (solve.hpp:133-142): every iteration's
/// detections go to on_detection before that iteration's sink.
template <SystemModel D, typename Sink, typename StepObs, typename DetObs>
void solve_iteratively(SolverBatch& batch, const D& def, const SolverConfig& cfg, Index iterations, Sink&& sink,
                       SolveObservers<StepObs, DetObs> observers) {
    if (iterations < 1) throw std::invalid_argument("solve_iteratively: iterations must be >= 1");
    for (Index i = 0; i < iterations; ++i) {
        solve(batch, def, cfg, observers);
        sink(i, static_cast<const SolverBatch&>(batch));
    }
}

/// Iterations back to back on the device, no host round trip (transient
/// iterations of a scan).
template <SystemModel D>
void solve_iteratively(SolverBatch& batch, const D& def, const SolverConfig& cfg, Index iterations) {
    if (iterations < 1) throw std::invalid_argument("solve_iteratively: iterations must be >= 1");
    if constexpr (BuiltinModel<D>) {
        detail::solve_iteratively_builtin<D, detail::NoSink>(batch, def, cfg, iterations, nullptr);
    } else {
        for (Index i = 0; i < iterations; ++i) solve_custom(batch, def, cfg);
    }
}

} // namespace odegpu

#endif
