// ref_harness.cpp — TEST INFRASTRUCTURE ONLY (oracle). Never linked into the
// product. Wraps the UNMODIFIED reference `odensemble::solve_iteratively`
// (/root/reference/proj/include/odensemble/solve.hpp:133-142) behind the
// same C structs the product ABI uses (include/odegpu.h), so tests, golden
// fixture generation and bench.py's CPU arm can drive the reference on SoA
// arrays. Built by oracle/Makefile into oracle/_ref/libodref.so from the
// reference sources where they lie (no copy).
//
// The reference's test fakes (RampDef, DecayDef, ...) are restated here as
// SystemModel types so their known answers can be replayed on the GPU path.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <exception>
#include <limits>
#include <span>
#include <string>

#include "odegpu.h"
#include "odensemble/models/duffing.hpp"
#include "odensemble/models/keller_miksis.hpp"
#include "odensemble/models/valve.hpp"
#include "odensemble/scan.hpp"
#include "odensemble/solve.hpp"

using namespace odensemble;

static_assert(sizeof(SystemOutcome) == sizeof(odegpu_outcome), "outcome layout");
static_assert(offsetof(odegpu_outcome, smallest_step) == offsetof(SystemOutcome, smallest_step));
static_assert(offsetof(odegpu_outcome, accepted_steps) == offsetof(SystemOutcome, accepted_steps));

namespace {

thread_local std::string g_err;

// cfg1 harness model: per-period running max and min of y1
// with their times, seeded from the initial state.
struct DuffingMaxMin : HookDefaults {
    OdeControls ode;
    SystemDims dims() const { return {2, 4, 0, 4}; }
    OdeControls ode_controls() const { return ode; }
    void ode_rhs(Real t, std::span<const Real> y, std::span<const Real> p, std::span<Real> dy) const {
        models::duffing_rhs(t, y, p, dy);
    }
    void initialize(Real t, std::span<Real>, std::span<Real> y, std::span<const Real>,
                    std::span<Real> acc) const {
        acc[0] = y[0];
        acc[1] = t;
        acc[2] = y[0];
        acc[3] = t;
    }
    void ordinary_accessory(Real t, std::span<const Real> y, std::span<const Real>,
                            std::span<Real> acc) const {
        if (y[0] > acc[0]) {
            acc[0] = y[0];
            acc[1] = t;
        }
        if (y[0] < acc[2]) {
            acc[2] = y[0];
            acc[3] = t;
        }
    }
};

struct OneDim : HookDefaults {
    OdeControls ode;
    OdeControls ode_controls() const { return ode; }
};

struct ConstantDef : OneDim {
    Real value = 0;
    SystemDims dims() const { return {1, 0, 0, 0}; }
    void ode_rhs(Real, std::span<const Real>, std::span<const Real>, std::span<Real> dy) const { dy[0] = value; }
};
struct CubicTimeDef : OneDim {
    SystemDims dims() const { return {1, 0, 0, 0}; }
    void ode_rhs(Real t, std::span<const Real>, std::span<const Real>, std::span<Real> dy) const {
        dy[0] = t * t * t;
    }
};
struct ExponentialDef : OneDim {
    SystemDims dims() const { return {1, 0, 0, 0}; }
    void ode_rhs(Real, std::span<const Real> y, std::span<const Real>, std::span<Real> dy) const { dy[0] = y[0]; }
};
struct UnitSlopeDef : OneDim {
    SystemDims dims() const { return {1, 0, 0, 0}; }
    void ode_rhs(Real, std::span<const Real>, std::span<const Real>, std::span<Real> dy) const { dy[0] = 1.0; }
};
struct BlowUpDef : OneDim {
    SystemDims dims() const { return {1, 0, 0, 0}; }
    void ode_rhs(Real, std::span<const Real>, std::span<const Real>, std::span<Real> dy) const {
        dy[0] = std::numeric_limits<Real>::quiet_NaN();
    }
};
struct CountingDef : OneDim {
    SystemDims dims() const { return {2, 4, 0, 3}; }
    void ode_rhs(Real t, std::span<const Real> y, std::span<const Real> p, std::span<Real> dy) const {
        models::duffing_rhs(t, y, p, dy);
    }
    void initialize(Real, std::span<Real>, std::span<Real>, std::span<const Real>, std::span<Real> acc) const {
        acc[0] += 1;
    }
    void finalize(Real, std::span<Real>, std::span<Real>, std::span<const Real>, std::span<Real> acc) const {
        acc[1] += 1;
    }
    void ordinary_accessory(Real, std::span<const Real>, std::span<const Real>, std::span<Real> acc) const {
        acc[2] += 1;
    }
};
struct RampDef : OneDim {
    Real slope = 1.0, level = 0.0, tol = 1e-6;
    int direction = 0;
    Index stop = 0, max_zone_steps = 50;
    SystemDims dims() const { return {1, 0, 1, 0}; }
    EventControls event_controls() const {
        return {.direction = {direction}, .tolerance = {tol}, .stop_condition = {stop},
                .max_steps_in_zone = max_zone_steps};
    }
    void ode_rhs(Real, std::span<const Real>, std::span<const Real>, std::span<Real> dy) const { dy[0] = slope; }
    void event_values(Real, std::span<const Real> y, std::span<const Real>, std::span<Real> f) const {
        f[0] = y[0] - level;
    }
};
struct DecayDef : OneDim {
    SystemDims dims() const { return {1, 0, 1, 0}; }
    EventControls event_controls() const {
        return {.direction = {0}, .tolerance = {1e-6}, .stop_condition = {0}, .max_steps_in_zone = 50};
    }
    void ode_rhs(Real, std::span<const Real> y, std::span<const Real>, std::span<Real> dy) const { dy[0] = -y[0]; }
    void event_values(Real, std::span<const Real> y, std::span<const Real>, std::span<Real> f) const { f[0] = y[0]; }
};
struct SeatContactDef : OneDim {
    SystemDims dims() const { return {3, 5, 1, 0}; }
    EventControls event_controls() const {
        return {.direction = {-1}, .tolerance = {1e-6}, .stop_condition = {1}};
    }
    void ode_rhs(Real t, std::span<const Real> y, std::span<const Real> p, std::span<Real> dy) const {
        models::valve_rhs(t, y, p, dy);
    }
    void event_values(Real, std::span<const Real> y, std::span<const Real>, std::span<Real> f) const { f[0] = y[0]; }
};
struct HarmonicDef : OneDim {
    SystemDims dims() const { return {2, 0, 0, 0}; }
    void ode_rhs(Real, std::span<const Real> y, std::span<const Real>, std::span<Real> dy) const {
        dy[0] = y[1];
        dy[1] = -y[0];
    }
};

struct Trace {
    double* td;
    double* state;
    double* acc;
    odegpu_outcome* outcomes;
};

// Detection capture (odref_capture_detections): the reference's own
// on_detection observer (solve.hpp:46-50) records every detection of the
// LAST solve of a run, per system in call order.
struct RefDetection {
    Index event_index, counter;
    double t, value;
    int kind, in_zone;
    std::vector<double> y_pre, y_post;
};
bool g_capture = false;
std::vector<std::vector<RefDetection>> g_dets;

template <SystemModel D>
int run(const D& def, Index n, double* td, double* y, const double* p, double* acc, odegpu_outcome* outcomes,
        int keep_outcomes, const SolverConfig& cfg, Index iterations, const Trace* trace, double* seconds) {
    const SystemDims sd = def.dims();
    ProblemPool pool(PoolDims{n, sd.system_dim, sd.param_count, sd.accessory_count});
    std::copy_n(td, 2 * n, pool.time_domain().begin());
    std::copy_n(y, sd.system_dim * n, pool.state().begin());
    if (sd.param_count) std::copy_n(p, sd.param_count * n, pool.parameters().begin());
    if (sd.accessory_count) std::copy_n(acc, sd.accessory_count * n, pool.accessories().begin());

    SolverBatch batch(make_batch_dims(n, sd));
    linear_set(batch, pool, LinearCopySpec{0, 0, n, CopyMode::All});
    if (keep_outcomes)
        std::memcpy(static_cast<void*>(batch.outcomes().data()), outcomes, sizeof(odegpu_outcome) * n);

    const auto t0 = std::chrono::steady_clock::now();
    if (g_capture) g_dets.assign(static_cast<std::size_t>(n), {});
    auto on_detection = [](Index s, const Detection& d, std::span<const Real> pre, std::span<const Real> post) {
        // workers own disjoint systems: one vector per system needs no lock
        g_dets[static_cast<std::size_t>(s)].push_back(RefDetection{d.event_index, d.counter, d.t, d.value,
                                                                   static_cast<int>(d.kind), d.in_zone ? 1 : 0,
                                                                   {pre.begin(), pre.end()},
                                                                   {post.begin(), post.end()}});
    };
    auto sink = [&](Index it, const SolverBatch& b) {
        if (g_capture && it + 1 < iterations) g_dets.assign(static_cast<std::size_t>(n), {}); // keep the last solve's
        if (!trace) return;
        const auto off = static_cast<std::size_t>(it);
        if (trace->td) std::copy(b.time_domain().begin(), b.time_domain().end(), trace->td + off * 2 * n);
        if (trace->state)
            std::copy(b.state().begin(), b.state().end(), trace->state + off * sd.system_dim * n);
        if (trace->acc && sd.accessory_count)
            std::copy(b.accessories().begin(), b.accessories().end(), trace->acc + off * sd.accessory_count * n);
        if (trace->outcomes)
            std::memcpy(static_cast<void*>(trace->outcomes + off * n), b.outcomes().data(),
                        sizeof(odegpu_outcome) * n);
    };
    if (g_capture)
        solve_iteratively(batch, def, cfg, iterations, sink,
                          SolveObservers<NoBatchStepObserver, decltype(on_detection)>{{}, on_detection});
    else
        solve_iteratively(batch, def, cfg, iterations, sink);
    const auto t1 = std::chrono::steady_clock::now();
    if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();

    std::copy(batch.time_domain().begin(), batch.time_domain().end(), td);
    std::copy(batch.state().begin(), batch.state().end(), y);
    if (sd.accessory_count) std::copy(batch.accessories().begin(), batch.accessories().end(), acc);
    std::memcpy(static_cast<void*>(outcomes), batch.outcomes().data(), sizeof(odegpu_outcome) * n);
    return 0;
}

OdeControls to_ode(Index dim, const odegpu_ode_controls* c) {
    OdeControls o;
    o.rel_tol.assign(c->rel_tol, c->rel_tol + dim);
    o.abs_tol.assign(c->abs_tol, c->abs_tol + dim);
    o.max_step = c->max_step;
    o.min_step = c->min_step;
    o.step_grow_limit = c->step_grow_limit;
    o.step_shrink_limit = c->step_shrink_limit;
    return o;
}

template <typename T>
T with_ode(Index dim, const odegpu_ode_controls* c) {
    T d;
    d.ode = to_ode(dim, c);
    return d;
}

} // namespace

extern "C" {

const char* odref_last_error(void) { return g_err.c_str(); }

// Turns the detection capture of odref_solve on (1) or off (0).
void odref_capture_detections(int on) {
    g_capture = on != 0;
    if (!g_capture) g_dets.clear();
}

// The captured detections of the last odref_solve in (system, call) order,
// in the C ABI's record layout (odegpu_detection) with system_dim doubles
// each of y_pre / y_post; returns the number available, writes <= capacity.
odegpu_index odref_detections(odegpu_detection* out, double* y_pre, double* y_post, odegpu_index capacity) {
    odegpu_index k = 0, total = 0;
    for (std::size_t s = 0; s < g_dets.size(); ++s) {
        for (std::size_t q = 0; q < g_dets[s].size(); ++q, ++total) {
            if (k >= capacity || !out) continue;
            const RefDetection& d = g_dets[s][q];
            out[k] = odegpu_detection{static_cast<odegpu_index>(s), d.event_index, d.counter,
                                      static_cast<odegpu_index>(q), d.t, d.value, d.kind, d.in_zone};
            const std::size_t dim = d.y_pre.size();
            for (std::size_t j = 0; j < dim; ++j) {
                if (y_pre) y_pre[static_cast<std::size_t>(k) * dim + j] = d.y_pre[j];
                if (y_post) y_post[static_cast<std::size_t>(k) * dim + j] = d.y_post[j];
            }
            ++k;
        }
    }
    return total;
}

// Runs `iterations` reference solves over n systems held in SoA arrays
// (td, y, acc updated in place; outcomes written). keep_outcomes != 0 seeds
// the batch outcomes from `outcomes` (sticky NonFiniteAbort, solve.hpp:98).
// trace_* (each nullable) receive per-iteration snapshots. *seconds gets the
// steady_clock time of solve_iteratively alone.
int odref_solve(const odegpu_model* m, odegpu_index n, double* td, double* y, const double* p, double* acc,
                odegpu_outcome* outcomes, int keep_outcomes, const odegpu_solver_config* c,
                const odegpu_ode_controls* ode, odegpu_index iterations, double* trace_td, double* trace_state,
                double* trace_acc, odegpu_outcome* trace_outcomes, double* seconds) {
    try {
        SolverConfig cfg;
        cfg.algorithm = c->algorithm == ODEGPU_RK4 ? Algorithm::RK4 : Algorithm::RKCK45;
        cfg.initial_time_step = c->initial_time_step;
        cfg.tile_size = c->tile_size;
        cfg.worker_count = c->worker_count;
        const Trace tr{trace_td, trace_state, trace_acc, trace_outcomes};
        const Trace* trp = (trace_td || trace_state || trace_acc || trace_outcomes) ? &tr : nullptr;
        const double* k = m->consts;
        auto go = [&](const auto& def) {
            return run(def, n, td, y, p, acc, outcomes, keep_outcomes, cfg, iterations, trp, seconds);
        };
        switch (m->id) {
        case ODEGPU_MODEL_DUFFING: return go(models::DuffingSystem(to_ode(2, ode)));
        case ODEGPU_MODEL_DUFFING_MAX_ACCESSORY: return go(models::DuffingMaxAccessorySystem(to_ode(2, ode)));
        case ODEGPU_MODEL_DUFFING_MAX_EVENT:
            return go(models::DuffingMaxEventSystem(k[0], static_cast<Index>(k[1]), to_ode(2, ode)));
        case ODEGPU_MODEL_DUFFING_MAXMIN: return go(with_ode<DuffingMaxMin>(2, ode));
        case ODEGPU_MODEL_KELLER_MIKSIS: return go(models::KellerMiksisSystem(to_ode(2, ode)));
        case ODEGPU_MODEL_BUBBLE_COLLAPSE: return go(models::BubbleCollapseSystem(k[0], to_ode(2, ode)));
        case ODEGPU_MODEL_VALVE: return go(models::ValveSystem(k[0], to_ode(3, ode)));
        case ODEGPU_MODEL_DUFFING_LYAPUNOV: return go(models::DuffingLyapunovSystem(to_ode(4, ode)));
        case ODEGPU_MODEL_CONSTANT: {
            auto d = with_ode<ConstantDef>(1, ode);
            d.value = k[0];
            return go(d);
        }
        case ODEGPU_MODEL_CUBIC_TIME: return go(with_ode<CubicTimeDef>(1, ode));
        case ODEGPU_MODEL_EXPONENTIAL: return go(with_ode<ExponentialDef>(1, ode));
        case ODEGPU_MODEL_UNIT_SLOPE: return go(with_ode<UnitSlopeDef>(1, ode));
        case ODEGPU_MODEL_COUNTING: return go(with_ode<CountingDef>(2, ode));
        case ODEGPU_MODEL_RAMP: {
            auto d = with_ode<RampDef>(1, ode);
            d.slope = k[0];
            d.level = k[1];
            d.direction = static_cast<int>(k[2]);
            d.stop = static_cast<Index>(k[3]);
            d.tol = k[4];
            d.max_zone_steps = static_cast<Index>(k[5]);
            return go(d);
        }
        case ODEGPU_MODEL_DECAY: return go(with_ode<DecayDef>(1, ode));
        case ODEGPU_MODEL_SEAT_CONTACT: return go(with_ode<SeatContactDef>(3, ode));
        case ODEGPU_MODEL_HARMONIC: return go(with_ode<HarmonicDef>(2, ode));
        case ODEGPU_MODEL_BLOWUP: return go(with_ode<BlowUpDef>(1, ode));
        default: g_err = "odref_solve: unknown model"; return ODEGPU_ERR_UNSUPPORTED;
        }
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return ODEGPU_ERR_INVALID_ARGUMENT;
    } catch (const std::out_of_range& e) {
        g_err = e.what();
        return ODEGPU_ERR_OUT_OF_RANGE;
    } catch (const std::exception& e) {
        g_err = e.what();
        return ODEGPU_ERR_CUDA;
    }
}

// bubble_coefficients (models/keller_miksis.hpp:47-77) for n grid points:
// phys[13*i + k] = BubblePhysical fields in declaration order; out[i + c*n].
int odref_bubble_coefficients(odegpu_index n, const double* phys, double* out) {
    try {
        for (Index i = 0; i < n; ++i) {
            const double* f = phys + 13 * i;
            models::BubblePhysical b{f[0], f[1], f[2], f[3], f[4], f[5], f[6],
                                     f[7], f[8], f[9], f[10], f[11], f[12]};
            const auto c = models::bubble_coefficients(b);
            for (Index k = 0; k < 13; ++k) out[i + k * n] = c[static_cast<std::size_t>(k)];
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return ODEGPU_ERR_INVALID_ARGUMENT;
    }
}

// scan::ParamRange::values (src/scan.cpp:17-37) -> out[res].
int odref_param_range(double lo, double hi, odegpu_index res, int log_scale, double* out) {
    try {
        scan::ParamRange r{lo, hi, res, log_scale ? scan::Scale::Log : scan::Scale::Linear};
        const auto v = r.values();
        std::copy(v.begin(), v.end(), out);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return ODEGPU_ERR_INVALID_ARGUMENT;
    }
}

// The reference's scan protocols (src/scan.cpp:145-370) on the same C specs
// as odegpu_scan_run (include/odegpu.h): rows row-major, diagnostics.
static scan::ParamRange ref_range(const odegpu_param_range& r) {
    return scan::ParamRange{r.min, r.max, r.res, r.log_scale ? scan::Scale::Log : scan::Scale::Linear};
}
static scan::SolveOptions ref_options(const odegpu_scan_options& o, int workers) {
    scan::SolveOptions s;
    s.algorithm = o.algorithm == ODEGPU_RK4 ? Algorithm::RK4 : Algorithm::RKCK45;
    s.dt = o.dt;
    s.rel_tol = o.rel_tol;
    s.abs_tol = o.abs_tol;
    s.event_tol = o.event_tol;
    s.batch_capacity = o.batch_capacity;
    s.workers = workers;
    return s;
}

int odref_scan_run(int32_t protocol, const void* spec, double* rows, odegpu_index max_rows, odegpu_index* n_rows,
                   odegpu_index* n_columns, odegpu_scan_diagnostics* diag, int workers) {
    try {
        scan::ScanResult r;
        if (protocol <= ODEGPU_SCAN_DUFFING_LYAPUNOV) {
            const auto& d = *static_cast<const odegpu_duffing_scan*>(spec);
            scan::DuffingScanSpec s;
            s.k = ref_range(d.k);
            s.forcing_amplitude = d.forcing_amplitude;
            s.stiffness = d.stiffness;
            s.forcing_omega = d.forcing_omega;
            s.ic = {d.ic[0], d.ic[1]};
            s.transient = d.transient;
            s.saved = d.saved;
            s.solver = ref_options(d.solver, workers);
            if (protocol == ODEGPU_SCAN_DUFFING_POINCARE) r = scan::run_duffing_poincare(s);
            else if (protocol == ODEGPU_SCAN_DUFFING_LYAPUNOV) r = scan::run_duffing_lyapunov(s);
            else
                r = scan::run_duffing_maxima(s, protocol == ODEGPU_SCAN_DUFFING_MAXIMA_EVENT ? scan::MaximaMode::Event
                                                                                              : scan::MaximaMode::Accessory);
        } else if (protocol == ODEGPU_SCAN_BUBBLE) {
            const auto& b = *static_cast<const odegpu_bubble_scan*>(spec);
            scan::BubbleScanSpec s;
            s.pa1_bar = ref_range(b.pa1_bar);
            s.pa2_bar = ref_range(b.pa2_bar);
            s.f1_khz = ref_range(b.f1_khz);
            s.f2_khz = ref_range(b.f2_khz);
            s.material.R_E = b.R_E;
            s.material.c_L = b.c_L;
            s.material.rho_L = b.rho_L;
            s.material.P_inf = b.P_inf;
            s.material.p_V = b.p_V;
            s.material.sigma = b.sigma;
            s.material.mu_L = b.mu_L;
            s.material.gamma = b.gamma;
            s.material.theta = b.theta;
            s.ic = {b.ic[0], b.ic[1]};
            s.t_end = b.t_end;
            s.transient = b.transient;
            s.saved = b.saved;
            s.solver = ref_options(b.solver, workers);
            r = scan::run_bubble_scan(s);
        } else if (protocol == ODEGPU_SCAN_VALVE) {
            const auto& v = *static_cast<const odegpu_valve_scan*>(spec);
            scan::ValveScanSpec s;
            s.q = ref_range(v.q);
            s.kappa = v.kappa;
            s.delta = v.delta;
            s.beta = v.beta;
            s.restitution = v.restitution;
            s.ic = {v.ic[0], v.ic[1], v.ic[2]};
            s.t_end = v.t_end;
            s.transient = v.transient;
            s.saved = v.saved;
            s.solver = ref_options(v.solver, workers);
            r = scan::run_valve_scan(s);
        } else {
            g_err = "scan: unknown protocol";
            return ODEGPU_ERR_INVALID_ARGUMENT;
        }
        const odegpu_index nr = std::ssize(r.rows), nc = std::ssize(r.columns);
        *n_rows = nr;
        *n_columns = nc;
        if (rows) {
            if (max_rows < nr) {
                g_err = "scan: rows buffer too small";
                return ODEGPU_ERR_OUT_OF_RANGE;
            }
            for (odegpu_index i = 0; i < nr; ++i)
                std::memcpy(rows + i * nc, r.rows[static_cast<std::size_t>(i)].data(), size_t(nc) * 8);
        }
        if (diag) {
            const auto& d = r.diagnostics;
            *diag = odegpu_scan_diagnostics{};
            diag->detections = d.detections;
            diag->detections_outside_zone = d.detections_outside_zone;
            diag->max_residual_ratio = d.max_residual_ratio;
            diag->secant_failures = d.secant_failures;
            diag->nonfinite_systems = d.nonfinite_systems;
            for (int k = 0; k < 4; ++k) diag->reason_counts[k] = d.reason_counts[static_cast<std::size_t>(k)];
            diag->start_times_strictly_increase = d.start_times_strictly_increase ? 1 : 0;
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return ODEGPU_ERR_INVALID_ARGUMENT;
    }
}

} // extern "C"
