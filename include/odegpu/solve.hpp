// solve.hpp — the drop-in entry points of the C++ host API:
// solve (/root/reference/proj/include/odensemble/solve.hpp:60-128) and
// solve_iteratively (solve.hpp:133-142), running on the GPU through the C ABI.
//
// Validation and its messages are the reference's (performed in libodegpu);
// failures are rethrown as std::invalid_argument / std::out_of_range.
// solve() is synchronous like the reference. Host observers are not
// supported on the device; per-solve tallies come from
// SolverBatch diagnostics instead.
#ifndef ODEGPU_SOLVE_HPP
#define ODEGPU_SOLVE_HPP

#include <exception>
#include <type_traits>
#include <stdexcept>
#include <utility>
#include <vector>

#include "odegpu.h"
#include "odegpu/batch.hpp"
#include "odegpu/system.hpp"

namespace odegpu {

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
