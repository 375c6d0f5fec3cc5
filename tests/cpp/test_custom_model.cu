// test_custom_model.cu — the SystemModel plugin path: models written by a
// user (not built into libodegpu), compiled by nvcc in this translation unit
// through include/odegpu/device/custom.cuh, solved with the same odegpu::solve
// calls as the built-in models. Exit code = failed checks.
#include <cmath>
#include <cstdio>
#include <numbers>
#include <span>
#include <string>
#include <vector>

#include "odegpu/device/custom.cuh"
#include "odegpu/odegpu.hpp"

using namespace odegpu;

static int g_checks = 0, g_failed = 0;
#define CHECK(cond)                                                                       \
    do {                                                                                  \
        ++g_checks;                                                                       \
        if (!(cond)) {                                                                    \
            ++g_failed;                                                                   \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);                   \
        }                                                                                 \
    } while (0)

constexpr Real kTwoPi = 2.0 * std::numbers::pi_v<Real>;

// A user's own restatement of DuffingMaxEventSystem (duffing.hpp:122-156).
struct MyDuffingHooks : HookDefaults {
    static constexpr Index kSystemDim = 2, kParamCount = 4, kEventCount = 1, kAccessoryCount = 2;
    ODEGPU_HD void ode_rhs(Real t, std::span<const Real> y, std::span<const Real> p, std::span<Real> dy) const {
        models::duffing_rhs(t, y, p, dy);
    }
    ODEGPU_HD void event_values(Real, std::span<const Real> y, std::span<const Real>, std::span<Real> f) const {
        f[0] = y[1];
    }
    ODEGPU_HD void initialize(Real t, std::span<Real>, std::span<Real> y, std::span<const Real>,
                              std::span<Real> acc) const {
        acc[0] = y[0];
        acc[1] = t;
    }
    ODEGPU_HD void event_accessory(Index e, Index, Real t, std::span<const Real> y, std::span<const Real>,
                                   std::span<Real> acc) const {
        if (e == 0 && y[0] > acc[0]) {
            acc[0] = y[0];
            acc[1] = t;
        }
    }
};
class MyDuffing : public MyDuffingHooks {
public:
    using hooks_type = MyDuffingHooks;
    SystemDims dims() const { return dims_of<hooks_type>(); }
    OdeControls ode_controls() const { return OdeControls::uniform(2, 1e-9, 1e-9); }
    EventControls event_controls() const { return {.direction = {-1}, .tolerance = {1e-6}, .stop_condition = {0}}; }
};

// A model the library has never seen: forced damped pendulum, the event
// theta' = 0 (falling) stops at the first turning point; hook data (gamma)
// lives in the hooks struct and travels in the kernel parameter bank.
struct PendulumHooks : HookDefaults {
    static constexpr Index kSystemDim = 2, kParamCount = 2, kEventCount = 1, kAccessoryCount = 1;
    Real gamma = 0.1;
    ODEGPU_HD void ode_rhs(Real t, std::span<const Real> y, std::span<const Real> p, std::span<Real> dy) const {
        dy[0] = y[1];
        dy[1] = -sin(y[0]) - gamma * y[1] + p[0] * cos(p[1] * t);
    }
    ODEGPU_HD void event_values(Real, std::span<const Real> y, std::span<const Real>, std::span<Real> f) const {
        f[0] = y[1];
    }
    ODEGPU_HD void ordinary_accessory(Real, std::span<const Real> y, std::span<const Real>,
                                      std::span<Real> acc) const {
        acc[0] = fmax(acc[0], fabs(y[0]));
    }
};
class Pendulum : public PendulumHooks {
public:
    using hooks_type = PendulumHooks;
    explicit Pendulum(Real g) { gamma = g; }
    SystemDims dims() const { return dims_of<hooks_type>(); }
    OdeControls ode_controls() const { return OdeControls::uniform(2, 1e-10, 1e-10); }
    EventControls event_controls() const { return {.direction = {-1}, .tolerance = {1e-8}, .stop_condition = {1}}; }
};

int main() {
    // 1. the clone equals the built-in model bit for bit
    const Index n = 512;
    ProblemPool pool(PoolDims{n, 2, 4, 2});
    for (Index i = 0; i < n; ++i) {
        pool.time_end(i) = kTwoPi;
        pool.param_at(i, 0) = 0.2 + 0.1 * static_cast<Real>(i) / (n - 1);
        pool.param_at(i, 1) = 0.3;
        pool.param_at(i, 2) = 1.0;
        pool.param_at(i, 3) = 1.0;
    }
    models::DuffingMaxEventSystem builtin(1e-6, 0);
    MyDuffing mine;
    SolverBatch a(make_batch_dims(n, builtin.dims())), b(make_batch_dims(n, mine.dims()));
    linear_set(a, pool, {0, 0, n, CopyMode::All});
    linear_set(b, pool, {0, 0, n, CopyMode::All});
    solve_iteratively(a, builtin, SolverConfig{}, 2);
    Index sink_calls = 0;
    solve_iteratively(b, mine, SolverConfig{}, 2, [&](Index, const SolverBatch&) { ++sink_calls; });
    CHECK(sink_calls == 2);
    const SolverBatch &ca = a, &cb = b;
    bool same = true;
    for (std::size_t k = 0; k < ca.state().size(); ++k) same = same && ca.state()[k] == cb.state()[k];
    for (std::size_t k = 0; k < ca.accessories().size(); ++k)
        same = same && ca.accessories()[k] == cb.accessories()[k];
    for (Index i = 0; i < n; ++i) {
        const auto &oa = ca.outcomes()[static_cast<std::size_t>(i)], &ob = cb.outcomes()[static_cast<std::size_t>(i)];
        same = same && oa.accepted_steps == ob.accepted_steps && oa.rejected_steps == ob.rejected_steps &&
               oa.event_detections == ob.event_detections && oa.final_t == ob.final_t;
    }
    CHECK(same);

    // 2. a new model: every system stops at its first turning point
    const Index m = 256;
    ProblemPool pp(PoolDims{m, 2, 2, 1});
    for (Index i = 0; i < m; ++i) {
        pp.time_end(i) = 100.0;
        pp.state_at(i, 1) = 0.5 + static_cast<Real>(i) / m; // initial angular velocity
        pp.param_at(i, 0) = 0.2;
        pp.param_at(i, 1) = 0.8;
    }
    Pendulum pend(0.1);
    SolverBatch pb(make_batch_dims(m, pend.dims()));
    linear_set(pb, pp, {0, 0, m, CopyMode::All});
    solve(pb, pend, SolverConfig{});
    const SolverBatch& cp = pb;
    for (Index i = 0; i < m; ++i) {
        CHECK(cp.outcomes()[static_cast<std::size_t>(i)].reason == StopReason::EventStop);
        CHECK(std::abs(cp.state_at(i, 1)) <= 1e-8);
        CHECK(cp.accessory_at(i, 0) >= std::abs(cp.state_at(i, 0)) - 1e-15);
    }

    // 3. validation and errors are the built-in ones
    bool threw = false;
    try {
        SolverConfig bad;
        bad.initial_time_step = -1;
        solve(pb, pend, bad);
    } catch (const std::invalid_argument& e) {
        threw = std::string(e.what()) == "solve: initial_time_step must be > 0";
    }
    CHECK(threw);

    std::printf("%d checks, %d failed\n", g_checks, g_failed);
    return g_failed;
}
