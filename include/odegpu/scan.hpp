// scan.hpp — the reference's experiment protocols (parameter sweeps with
// transient + saved iterations) on the GPU pipeline: same names, specs,
// result rows, diagnostics and CSV format as
// /root/reference/proj/include/odensemble/scan.hpp:14-134 and
// src/scan.cpp:17-400 — SURVEY.md §8f rows 1-2.
//
// What changes is run_chunks (src/scan.cpp:88-112): instead of one host
// sink call per iteration over host arrays, every chunk runs all its
// iterations back to back on the device (odegpu_pipeline, double-buffered
// H2D / solve / D2H); only the saved iterations' fields a protocol reads are
// copied back, and DiagCollector's per-iteration tallies are accumulated on
// the device (odegpu_scan_tally) — transient iterations never touch the host.
// Rows, statuses and diagnostics match the reference's (tests/test_gpu_scan.py).
//
// Header-only C++20 over the C ABI (plain g++ + libodegpu).
#ifndef ODEGPU_SCAN_HPP
#define ODEGPU_SCAN_HPP

#include <array>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <fstream>
#include <limits>
#include <numbers>
#include <stdexcept>
#include <string>
#include <vector>

#include "odegpu.h"
#include "odegpu/batch.hpp"
#include "odegpu/models/duffing.hpp"
#include "odegpu/models/keller_miksis.hpp"
#include "odegpu/models/valve.hpp"
#include "odegpu/pool.hpp"
#include "odegpu/solve.hpp"

namespace odegpu::scan {

enum class Scale { Linear, Log };

/// A scanned parameter axis; res = 1 yields just {min} (scan.cpp:17-37).
struct ParamRange {
    Real min = 0;
    Real max = 0;
    Index res = 1;
    Scale scale = Scale::Linear;

    std::vector<Real> values() const {
        if (res < 1) throw std::invalid_argument("ParamRange: res must be >= 1");
        if (res == 1) return {min};
        if (scale == Scale::Log && (!(min > 0) || !(max > 0)))
            throw std::invalid_argument("ParamRange: log scale requires positive bounds");
        std::vector<Real> out(static_cast<std::size_t>(res));
        for (Index i = 0; i < res; ++i) {
            if (i == 0) {
                out[0] = min;
            } else if (i == res - 1) {
                out[static_cast<std::size_t>(i)] = max;
            } else if (scale == Scale::Linear) {
                out[static_cast<std::size_t>(i)] = min + static_cast<Real>(i) * (max - min) / static_cast<Real>(res - 1);
            } else {
                out[static_cast<std::size_t>(i)] =
                    min * std::exp(static_cast<Real>(i) * std::log(max / min) / static_cast<Real>(res - 1));
            }
        }
        return out;
    }
};

/// Numerical settings shared by every scan (scan.hpp:29-38). workers and
/// tile_size are kept for source compatibility; the device schedules by
/// warps. batch_capacity = 0 solves the whole pool as one chunk.
struct SolveOptions {
    Algorithm algorithm = Algorithm::RKCK45;
    Real dt = 1e-3;
    Real rel_tol = 1e-9;
    Real abs_tol = 1e-9;
    Real event_tol = 1e-6;
    Index workers = 0;
    Index tile_size = 64;
    Index batch_capacity = 0;
    int device = 0;
    /// More than one entry: the chunks are spread over these devices (whole
    /// chunks, pool order — rows and diagnostics equal the one-device run's).
    std::vector<int> devices{};
};

/// scan.hpp:41-49
struct ScanDiagnostics {
    Index detections = 0;
    Index detections_outside_zone = 0;
    Real max_residual_ratio = 0;
    Index secant_failures = 0;
    Index nonfinite_systems = 0;
    std::array<Index, 4> reason_counts{};
    bool start_times_strictly_increase = true;
};

/// scan.hpp:53-57
struct ScanResult {
    std::vector<std::string> columns;
    std::vector<std::vector<Real>> rows;
    ScanDiagnostics diagnostics;
};

/// scan.hpp:59-69
struct DuffingScanSpec {
    ParamRange k{0.2, 0.3, 256, Scale::Linear};
    Real forcing_amplitude = 0.3;
    Real stiffness = 1.0;
    Real forcing_omega = 1.0;
    std::array<Real, 2> ic{0.0, 0.0};
    Index transient = 1024;
    Index saved = 32;
    SolveOptions solver{};
    std::string output;
};

enum class MaximaMode { Accessory, Event };

/// scan.hpp:73-87 (amplitudes in bar, frequencies in kHz)
struct BubbleScanSpec {
    ParamRange pa1_bar{1.1, 1.1, 1, Scale::Linear};
    ParamRange pa2_bar{0.7, 0.7, 1, Scale::Linear};
    ParamRange f1_khz{20.0, 1000.0, 32, Scale::Log};
    ParamRange f2_khz{20.0, 1000.0, 32, Scale::Log};
    models::BubblePhysical material{};
    std::array<Real, 2> ic{1.0, 0.0};
    Real t_end = 1e6;
    Index transient = 64;
    Index saved = 8;
    SolveOptions solver{.rel_tol = 1e-10, .abs_tol = 1e-10};
    std::string output;
};

/// scan.hpp:89-105
struct ValveScanSpec {
    ParamRange q{0.2, 10.0, 256, Scale::Linear};
    Real kappa = 1.25;
    Real delta = 10.0;
    Real beta = 20.0;
    Real restitution = 0.8;
    std::array<Real, 3> ic{0.2, 0.0, std::numeric_limits<Real>::quiet_NaN()};
    Real t_end = 1e6;
    Index transient = 256;
    Index saved = 32;
    SolveOptions solver{.rel_tol = 1e-10, .abs_tol = 1e-10};
    std::string output;
};

/// scan.hpp:128-134: "# " + comma-joined names, rows of %.16e.
inline void emit_rows(const std::string& path, const std::vector<std::string>& columns,
                      const std::vector<std::vector<Real>>& rows) {
    for (const auto& row : rows)
        if (row.size() != columns.size()) throw std::invalid_argument("emit_rows: row width does not match header");
    std::ofstream file(path);
    if (!file) throw std::runtime_error("emit_rows: cannot open '" + path + "' for writing");
    file << "# ";
    for (std::size_t i = 0; i < columns.size(); ++i) {
        if (i) file << ',';
        file << columns[i];
    }
    file << '\n';
    char buf[32];
    for (const auto& row : rows) {
        for (std::size_t i = 0; i < row.size(); ++i) {
            if (i) file << ',';
            std::snprintf(buf, sizeof(buf), "%.16e", row[i]);
            file << buf;
        }
        file << '\n';
    }
    if (!file) throw std::runtime_error("emit_rows: write to '" + path + "' failed");
}

namespace detail {

inline constexpr Real kTwoPi = 2.0 * std::numbers::pi_v<Real>;
inline constexpr uint32_t kRecTd = 1u, kRecState = 2u, kRecAcc = 8u, kRecOutcomes = 16u;

/// What a protocol's chunk sink sees: the saved iterations of one chunk.
struct Chunk {
    Index start = 0, count = 0, n_saved = 0;
    const odegpu_chunk_record* rec = nullptr;
    const odegpu_outcome* final_outcomes = nullptr; // after the chunk's last iteration
    Index system_dim = 0, accessory_count = 0;
    Real state(Index r, Index s, Index c) const { return rec->state[(r * system_dim + c) * count + s]; }
    Real acc(Index r, Index s, Index c) const { return rec->accessories[(r * accessory_count + c) * count + s]; }
    bool aborted(Index r, Index s) const {
        return rec->outcomes[r * count + s].reason == static_cast<uint8_t>(StopReason::NonFiniteAbort);
    }
    bool aborted_final(Index s) const {
        return final_outcomes[start + s].reason == static_cast<uint8_t>(StopReason::NonFiniteAbort);
    }
};

/// run_chunks (src/scan.cpp:88-112) on the device pipeline: the pool in
/// chunks of batch_capacity systems, transient + saved iterations per chunk,
/// on_chunk(Chunk, rows) with the saved iterations' records appends the
/// chunk's rows; chunks may finish out of order on several devices, so rows
/// are gathered per chunk and concatenated in pool order. The tallies go to
/// `diag`.
using Rows = std::vector<std::vector<Real>>;

/// ODEGPU_SCAN_TRACE=1: host-side phase times of a scan on stderr.
inline void scan_trace(const char* what) {
    static const bool on = std::getenv("ODEGPU_SCAN_TRACE") != nullptr;
    if (!on) return;
    static auto t0 = std::chrono::steady_clock::now();
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    std::fprintf(stderr, "[scan] %10.3f ms  %s\n", ms, what);
}

template <SystemModel D, class OnChunk>
void run_chunks(const D& def, const ProblemPool& pool, const SolveOptions& opt, Index transient, Index saved,
                uint32_t record_mask, ScanResult& result, OnChunk&& on_chunk, bool check_start_times = false) {
    const Index n_pool = pool.size();
    const Index cap = opt.batch_capacity > 0 ? std::min(opt.batch_capacity, n_pool) : n_pool;
    const SolverConfig cfg{opt.algorithm, opt.dt, opt.tile_size, opt.workers};
    odegpu::detail::CControls cc(def, cfg);
    const odegpu_model m = def.descriptor();
    std::vector<odegpu_outcome> final_outcomes(static_cast<std::size_t>(n_pool));
    odegpu_pool_out out{};
    out.outcomes = final_outcomes.data();
    std::vector<Rows> chunk_rows(static_cast<std::size_t>((n_pool + cap - 1) / cap));
    struct Ctx {
        OnChunk* f;
        const odegpu_outcome* fin;
        Index dim, acc, cap;
        std::vector<Rows>* rows;
        std::exception_ptr err;
    } ctx{&on_chunk, final_outcomes.data(), def.dims().system_dim, def.dims().accessory_count, cap, &chunk_rows,
          nullptr};
    // A chunk's final outcomes land in `out` before its sink runs (the
    // pipeline drains a slot — endpoint D2H first — then calls the sink).
    auto sink = [](odegpu_index start, odegpu_index count, odegpu_index n_rec, const odegpu_chunk_record* rec,
                   void* user) -> int {
        auto* c = static_cast<Ctx*>(user);
        try {
            (*c->f)(Chunk{start, count, n_rec, rec, c->fin, c->dim, c->acc},
                    (*c->rows)[static_cast<std::size_t>(start / c->cap)]);
        } catch (...) {
            c->err = std::current_exception();
            return ODEGPU_ERR_INVALID_ARGUMENT;
        }
        return 0;
    };
    odegpu_scan_tally t{};
    const odegpu_pool_view v = pool.view();
    int rc = 0;
    scan_trace("run_chunks: start");
    if (opt.devices.size() > 1) {
        rc = odegpu_solve_pool_multi_tallied(&v, &out, &m, &cc.c_cfg, &cc.c_ode, &cc.c_ev, cap, transient + saved,
                                             transient, record_mask | kRecOutcomes, sink, &ctx, opt.devices.data(),
                                             static_cast<int>(opt.devices.size()), 1, &t);
    } else {
        odegpu_pipeline* pipe = nullptr;
        odegpu::detail::check(odegpu_pipeline_create(&m, cap, opt.devices.empty() ? opt.device : opt.devices[0], &pipe));
        scan_trace("run_chunks: pipeline created");
        rc = odegpu_pipeline_run_tallied(pipe, &v, &out, &cc.c_cfg, &cc.c_ode, &cc.c_ev, transient + saved, transient,
                                         record_mask | kRecOutcomes, sink, &ctx, &t);
        scan_trace("run_chunks: pipeline run");
        odegpu_pipeline_destroy(pipe);
        scan_trace("run_chunks: pipeline destroyed");
    }
    if (ctx.err) std::rethrow_exception(ctx.err);
    odegpu::detail::check(rc);
    for (auto& r : chunk_rows)
        for (auto& row : r) result.rows.push_back(std::move(row));
    scan_trace("run_chunks: rows gathered");
    ScanDiagnostics& diag = result.diagnostics;
    diag.detections += t.detections;
    diag.detections_outside_zone += t.detections_outside_zone;
    diag.max_residual_ratio = std::max(diag.max_residual_ratio, t.max_residual_ratio);
    diag.secant_failures += t.secant_failures;
    diag.nonfinite_systems += t.nonfinite_systems;
    for (int r = 0; r < 4; ++r) diag.reason_counts[static_cast<std::size_t>(r)] += t.reason_counts[r];
    // only the bubble scan tracks it (src/scan.cpp:293-299)
    if (check_start_times && t.start_time_not_advanced) diag.start_times_strictly_increase = false;
}

inline Real status(bool aborted) { return aborted ? 1.0 : 0.0; }

inline void fill_duffing_pool(ProblemPool& pool, const DuffingScanSpec& spec, const std::vector<Real>& ks,
                              Index system_dim) {
    const Real period = kTwoPi / spec.forcing_omega;
    for (Index i = 0; i < pool.size(); ++i) {
        pool.time_start(i) = 0.0;
        pool.time_end(i) = period;
        pool.state_at(i, 0) = spec.ic[0];
        pool.state_at(i, 1) = spec.ic[1];
        if (system_dim == 4) {
            pool.state_at(i, 2) = 1.0; // linearized radius
            pool.state_at(i, 3) = 0.0; // linearized angle
        }
        models::DuffingParams p{ks[static_cast<std::size_t>(i)], spec.forcing_amplitude, spec.stiffness,
                                spec.forcing_omega};
        p.validate();
        std::array<Real, models::DuffingParams::count> buf{};
        p.write(buf);
        for (Index c = 0; c < models::DuffingParams::count; ++c) pool.param_at(i, c) = buf[static_cast<std::size_t>(c)];
    }
}

inline void maybe_emit(const ScanResult& r, const std::string& path) {
    if (!path.empty()) emit_rows(path, r.columns, r.rows);
}

} // namespace detail

/// scan.cpp:145-169 — columns k, B, y1, y2, status; one row per saved
/// iteration and system.
inline ScanResult run_duffing_poincare(const DuffingScanSpec& spec) {
    const auto ks = spec.k.values();
    ProblemPool pool(PoolDims{std::ssize(ks), 2, models::DuffingParams::count, 0});
    detail::fill_duffing_pool(pool, spec, ks, 2);
    models::DuffingSystem def(OdeControls::uniform(2, spec.solver.rel_tol, spec.solver.abs_tol));
    ScanResult result;
    result.columns = {"k", "B", "y1", "y2", "status"};
    detail::run_chunks(def, pool, spec.solver, spec.transient, spec.saved, detail::kRecState, result,
                       [&](const detail::Chunk& c, detail::Rows& rows) {
                           for (Index r = 0; r < c.n_saved; ++r)
                               for (Index s = 0; s < c.count; ++s)
                                   rows.push_back({ks[static_cast<std::size_t>(c.start + s)],
                                                          spec.forcing_amplitude, c.state(r, s, 0), c.state(r, s, 1),
                                                          detail::status(c.aborted(r, s))});
                       });
    detail::maybe_emit(result, spec.output);
    return result;
}

/// scan.cpp:171-203 — columns k, y1_max, status.
inline ScanResult run_duffing_maxima(const DuffingScanSpec& spec, MaximaMode mode) {
    const auto ks = spec.k.values();
    ProblemPool pool(PoolDims{std::ssize(ks), 2, models::DuffingParams::count, 2});
    detail::fill_duffing_pool(pool, spec, ks, 2);
    const OdeControls ode = OdeControls::uniform(2, spec.solver.rel_tol, spec.solver.abs_tol);
    ScanResult result;
    result.columns = {"k", "y1_max", "status"};
    const auto collect = [&](const auto& def) {
        detail::run_chunks(def, pool, spec.solver, spec.transient, spec.saved, detail::kRecAcc, result,
                           [&](const detail::Chunk& c, detail::Rows& rows) {
                               for (Index r = 0; r < c.n_saved; ++r)
                                   for (Index s = 0; s < c.count; ++s)
                                       rows.push_back({ks[static_cast<std::size_t>(c.start + s)],
                                                              c.acc(r, s, 0), detail::status(c.aborted(r, s))});
                           });
    };
    if (mode == MaximaMode::Accessory)
        collect(models::DuffingMaxAccessorySystem(ode));
    else
        collect(models::DuffingMaxEventSystem(spec.solver.event_tol, 0, ode));
    detail::maybe_emit(result, spec.output);
    return result;
}

/// scan.cpp:205-245 — columns k, lambda_max, status; lambda averaged over the
/// saved iterations (lyapunov_accumulate, duffing.hpp:62-71).
inline ScanResult run_duffing_lyapunov(const DuffingScanSpec& spec) {
    const auto ks = spec.k.values();
    const Real period = detail::kTwoPi / spec.forcing_omega;
    ProblemPool pool(PoolDims{std::ssize(ks), 4, models::DuffingParams::count, 1});
    detail::fill_duffing_pool(pool, spec, ks, 4);
    models::DuffingLyapunovSystem def(OdeControls::uniform(4, spec.solver.rel_tol, spec.solver.abs_tol));
    ScanResult result;
    result.columns = {"k", "lambda_max", "status"};
    detail::run_chunks(def, pool, spec.solver, spec.transient, spec.saved, detail::kRecAcc, result,
                       [&](const detail::Chunk& c, detail::Rows& rows) {
                           std::vector<Real> samples;
                           for (Index s = 0; s < c.count; ++s) {
                               samples.clear();
                               for (Index r = 0; r < c.n_saved; ++r)
                                   if (!c.aborted(r, s)) samples.push_back(c.acc(r, s, 0));
                               Real lambda = 0;
                               Real st = detail::status(c.aborted_final(s));
                               bool valid = !samples.empty();
                               for (Real v : samples) valid = valid && v > 0 && std::isfinite(v);
                               if (valid)
                                   lambda = models::lyapunov_accumulate(samples, period);
                               else
                                   st = 1.0;
                               rows.push_back({ks[static_cast<std::size_t>(c.start + s)], lambda, st});
                           }
                       });
    detail::maybe_emit(result, spec.output);
    return result;
}

/// scan.cpp:247-329 — columns omega1_radps, omega2_radps, pa1_pa, pa2_pa,
/// y_exp, status; y_exp = the largest relative expansion over the saved
/// collapses. The strictly increasing start-time check runs on the device.
inline ScanResult run_bubble_scan(const BubbleScanSpec& spec) {
    detail::scan_trace("bubble: start");
    const auto pa1s = spec.pa1_bar.values();
    const auto pa2s = spec.pa2_bar.values();
    const auto f1s = spec.f1_khz.values();
    const auto f2s = spec.f2_khz.values();
    struct GridPoint {
        Real pa1, pa2, w1, w2;
    };
    std::vector<GridPoint> grid;
    grid.reserve(pa1s.size() * pa2s.size() * f1s.size() * f2s.size());
    for (Real pa1 : pa1s)
        for (Real pa2 : pa2s)
            for (Real f1 : f1s)
                for (Real f2 : f2s)
                    grid.push_back({pa1 * 1e5, pa2 * 1e5, f1 * 1e3 * detail::kTwoPi, f2 * 1e3 * detail::kTwoPi});
    ProblemPool pool(PoolDims{std::ssize(grid), 2, models::BubbleCoefficients::count, 4});
    for (Index i = 0; i < pool.size(); ++i) {
        const GridPoint& g = grid[static_cast<std::size_t>(i)];
        models::BubblePhysical phys = spec.material;
        phys.pa1 = g.pa1;
        phys.pa2 = g.pa2;
        phys.omega1 = g.w1;
        phys.omega2 = g.w2;
        const auto coeff = models::bubble_coefficients(phys);
        for (Index c = 0; c < models::BubbleCoefficients::count; ++c)
            pool.param_at(i, c) = coeff[static_cast<std::size_t>(c)];
        pool.time_start(i) = 0.0;
        pool.time_end(i) = spec.t_end;
        pool.state_at(i, 0) = spec.ic[0];
        pool.state_at(i, 1) = spec.ic[1];
    }
    models::BubbleCollapseSystem def(spec.solver.event_tol,
                                     OdeControls::uniform(2, spec.solver.rel_tol, spec.solver.abs_tol));
    detail::scan_trace("bubble: pool filled");
    ScanResult result;
    result.columns = {"omega1_radps", "omega2_radps", "pa1_pa", "pa2_pa", "y_exp", "status"};
    detail::run_chunks(def, pool, spec.solver, spec.transient, spec.saved, detail::kRecAcc, result,
                       [&](const detail::Chunk& c, detail::Rows& rows) {
                           for (Index s = 0; s < c.count; ++s) {
                               Real yexp = -std::numeric_limits<Real>::infinity();
                               for (Index r = 0; r < c.n_saved; ++r)
                                   if (!c.aborted(r, s)) yexp = std::max(yexp, c.acc(r, s, 1) - 1.0);
                               Real st = detail::status(c.aborted_final(s));
                               if (!std::isfinite(yexp)) {
                                   yexp = 0.0;
                                   st = 1.0;
                               }
                               const GridPoint& g = grid[static_cast<std::size_t>(c.start + s)];
                               rows.push_back({g.w1, g.w2, g.pa1, g.pa2, yexp, st});
                           }
                       },
                       /*check_start_times=*/true);
    detail::maybe_emit(result, spec.output);
    return result;
}

/// scan.cpp:331-370 — columns q, y1_max, y1_min, status; one row per saved
/// iteration and system.
inline ScanResult run_valve_scan(const ValveScanSpec& spec) {
    const auto qs = spec.q.values();
    ProblemPool pool(PoolDims{std::ssize(qs), 3, models::ValveParams::count, 2});
    const Real ic_pressure = std::isnan(spec.ic[2]) ? spec.delta + 0.2 : spec.ic[2];
    for (Index i = 0; i < pool.size(); ++i) {
        models::ValveParams p{spec.kappa, spec.delta, spec.beta, qs[static_cast<std::size_t>(i)], spec.restitution};
        p.validate();
        std::array<Real, models::ValveParams::count> buf{};
        p.write(buf);
        for (Index c = 0; c < models::ValveParams::count; ++c) pool.param_at(i, c) = buf[static_cast<std::size_t>(c)];
        pool.time_start(i) = 0.0;
        pool.time_end(i) = spec.t_end;
        pool.state_at(i, 0) = spec.ic[0];
        pool.state_at(i, 1) = spec.ic[1];
        pool.state_at(i, 2) = ic_pressure;
    }
    models::ValveSystem def(spec.solver.event_tol, OdeControls::uniform(3, spec.solver.rel_tol, spec.solver.abs_tol));
    ScanResult result;
    result.columns = {"q", "y1_max", "y1_min", "status"};
    detail::run_chunks(def, pool, spec.solver, spec.transient, spec.saved, detail::kRecAcc, result,
                       [&](const detail::Chunk& c, detail::Rows& rows) {
                           for (Index r = 0; r < c.n_saved; ++r)
                               for (Index s = 0; s < c.count; ++s)
                                   rows.push_back({qs[static_cast<std::size_t>(c.start + s)], c.acc(r, s, 0),
                                                          c.acc(r, s, 1), detail::status(c.aborted(r, s))});
                       });
    detail::maybe_emit(result, spec.output);
    return result;
}

} // namespace odegpu::scan

#endif
