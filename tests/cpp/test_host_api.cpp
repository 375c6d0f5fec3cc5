// test_host_api.cpp — the reference test-suite's batch / driver / scan cases
// (/root/reference/proj/tests/test_{pool,batch,driver,scan}.cpp) written
// against the odegpu C++ host API, running on the GPU. Built by `make
// cpptests` (g++ only; links libodegpu.so) and driven by
// tests/test_gpu_cpp_api.py. Exit code = number of failed checks.
#include <cmath>
#include <cstdio>
#include <functional>
#include <limits>
#include <numbers>
#include <string>
#include <vector>

#include "odegpu/odegpu.hpp"
#include "odegpu/scan.hpp"

using namespace odegpu;

static int g_checks = 0, g_failed = 0;
static const char* g_case = "";

#define CHECK(cond)                                                                              \
    do {                                                                                         \
        ++g_checks;                                                                              \
        if (!(cond)) {                                                                           \
            ++g_failed;                                                                          \
            std::printf("FAIL [%s] %s:%d: %s\n", g_case, __FILE__, __LINE__, #cond);             \
        }                                                                                        \
    } while (0)

#define CHECK_THROWS_AS(expr, type)                                                              \
    do {                                                                                         \
        bool ok_ = false;                                                                        \
        try {                                                                                    \
            expr;                                                                                \
        } catch (const type&) {                                                                  \
            ok_ = true;                                                                          \
        } catch (...) {                                                                          \
        }                                                                                        \
        CHECK(ok_ && #type);                                                                     \
    } while (0)

static void run_case(const char* name, const std::function<void()>& f) {
    g_case = name;
    try {
        f();
    } catch (const std::exception& e) {
        ++g_failed;
        std::printf("FAIL [%s] unexpected exception: %s\n", name, e.what());
    }
}

constexpr Real kTwoPi = 2.0 * std::numbers::pi_v<Real>;

// test_system.cpp:16-38: a deliberately broken definition (declares two
// events, writes one) and a one-dimensional model with mutable controls.
struct ShortEventHooks : HookDefaults {
    static constexpr Index kSystemDim = 2, kParamCount = 0, kEventCount = 2, kAccessoryCount = 0;
    void ode_rhs(Real, std::span<const Real>, std::span<const Real>, std::span<Real> dy) const {
        dy[0] = 0;
        dy[1] = 0;
    }
    void event_values(Real, std::span<const Real> y, std::span<const Real>, std::span<Real> f) const {
        f[0] = y[0]; // f[1] forgotten
    }
};
struct ShortEventDef : ShortEventHooks {
    using hooks_type = ShortEventHooks;
    SystemDims dims() const { return {2, 0, 2, 0}; }
    OdeControls ode_controls() const { return OdeControls::uniform(2, 1e-9, 1e-9); }
    EventControls event_controls() const {
        return {.direction = {0, 0}, .tolerance = {1e-6, 1e-6}, .stop_condition = {0, 0}};
    }
};
struct OneDimHooks : HookDefaults {
    static constexpr Index kSystemDim = 1, kParamCount = 0, kEventCount = 0, kAccessoryCount = 0;
    void ode_rhs(Real, std::span<const Real>, std::span<const Real>, std::span<Real> dy) const { dy[0] = 0; }
};
struct ControlsDef : OneDimHooks {
    using hooks_type = OneDimHooks;
    OdeControls ode;
    SystemDims dims() const { return {1, 0, 0, 0}; }
    OdeControls ode_controls() const { return ode; }
    EventControls event_controls() const { return {}; }
};

static ProblemPool duffing_pool(Index n, Real k_lo = 0.2, Real k_hi = 0.3) { // test_batch.cpp:18-33
    ProblemPool pool(PoolDims{n, 2, 4, 0});
    for (Index i = 0; i < n; ++i) {
        pool.time_start(i) = 0.0;
        pool.time_end(i) = kTwoPi;
        const Real k = n == 1 ? k_lo : k_lo + (k_hi - k_lo) * static_cast<Real>(i) / static_cast<Real>(n - 1);
        models::DuffingParams{k, 0.3, 1.0, 1.0}.write(
            std::span<Real>(std::vector<Real>(4).data(), 4)); // exercise write()
        pool.param_at(i, 0) = k;
        pool.param_at(i, 1) = 0.3;
        pool.param_at(i, 2) = 1.0;
        pool.param_at(i, 3) = 1.0;
    }
    return pool;
}

int main() {
    run_case("linear_set round trip and single property", [] { // test_pool.cpp:69-107
        ProblemPool pool(PoolDims{16, 2, 4, 3});
        for (Index i = 0; i < 16; ++i) {
            pool.time_start(i) = 1000 + i;
            pool.time_end(i) = 2000 + i;
            for (Index c = 0; c < 2; ++c) pool.state_at(i, c) = 100 * c + i + 0.5;
            for (Index c = 0; c < 4; ++c) pool.param_at(i, c) = 10000 + 100 * c + i;
            for (Index c = 0; c < 3; ++c) pool.accessory_at(i, c) = -(100.0 * c + i) - 0.25;
        }
        SolverBatch all(BatchDims{16, 2, 4, 0, 3});
        linear_set(all, pool, {0, 0, 16, CopyMode::All});
        const SolverBatch& ca = all;
        for (Index i = 0; i < 16; ++i) {
            CHECK(ca.time_end(i) == pool.time_end(i));
            CHECK(ca.state_at(i, 1) == pool.state_at(i, 1));
            CHECK(ca.param_at(i, 3) == pool.param_at(i, 3));
            CHECK(ca.accessory_at(i, 2) == pool.accessory_at(i, 2));
        }
        SolverBatch part(BatchDims{8, 2, 4, 0, 3});
        linear_set(part, pool, {2, 5, 4, CopyMode::ActualState});
        const SolverBatch& cp = part;
        CHECK(cp.state_at(2, 0) == pool.state_at(5, 0));
        CHECK(cp.state_at(5, 1) == pool.state_at(8, 1));
        CHECK(cp.state_at(0, 0) == 0.0 && cp.state_at(6, 0) == 0.0);
        CHECK(cp.time_end(3) == 0.0 && cp.param_at(3, 0) == 0.0);
        CHECK_THROWS_AS(linear_set(part, pool, {4, 0, 5, CopyMode::All}), std::out_of_range);
        CHECK_THROWS_AS(linear_set(part, pool, {0, 12, 5, CopyMode::All}), std::out_of_range);
        SolverBatch wrong(BatchDims{8, 3, 4, 0, 3});
        CHECK_THROWS_AS(linear_set(wrong, pool, {0, 0, 2, CopyMode::All}), std::invalid_argument);
    });

    run_case("host writes through spans reach the device", [] {
        models::DuffingSystem def;
        SolverBatch b(make_batch_dims(2, def.dims()));
        auto td = b.time_domain();
        td[2] = kTwoPi; // t1 of system 0
        td[3] = kTwoPi;
        auto p = b.parameters();
        for (Index i = 0; i < 2; ++i) {
            p[static_cast<std::size_t>(0 * 2 + i)] = 0.25;
            p[static_cast<std::size_t>(1 * 2 + i)] = 0.3;
            p[static_cast<std::size_t>(2 * 2 + i)] = 1.0;
            p[static_cast<std::size_t>(3 * 2 + i)] = 1.0;
        }
        solve(b, def);
        const SolverBatch& cb = b;
        CHECK(cb.outcomes()[0].final_t == kTwoPi);
        CHECK(cb.outcomes()[1].accepted_steps > 10);
        CHECK(cb.state_at(0, 0) == cb.state_at(1, 0));
    });

    run_case("mutable spans held across solves stay live", [] {
        // the reference's spans point into live batch storage: a span taken
        // before solve() shows the solve's results and writes made through it
        // afterwards reach the next solve (they used to be lost)
        const auto pool = duffing_pool(4);
        models::DuffingSystem def;
        SolverBatch b(make_batch_dims(4, def.dims()));
        SolverBatch ref(make_batch_dims(4, def.dims()));
        linear_set(b, pool, {0, 0, 4, CopyMode::All});
        linear_set(ref, pool, {0, 0, 4, CopyMode::All});
        auto y = b.state(); // taken once, before any solve
        auto td = b.time_domain();
        solve(b, def);
        solve(ref, def);
        const SolverBatch& cr = ref;
        for (Index i = 0; i < 4; ++i) CHECK(y[static_cast<std::size_t>(i)] == cr.state_at(i, 0));
        // restart system 2 from the origin over [0, 2 pi] through the old spans
        y[2] = 0.0;
        y[2 + 4] = 0.0;
        td[2] = 0.0;
        td[2 + 4] = kTwoPi;
        solve(b, def);
        auto ry = ref.state();
        auto rtd = ref.time_domain();
        ry[2] = 0.0;
        ry[2 + 4] = 0.0;
        rtd[2] = 0.0;
        rtd[2 + 4] = kTwoPi;
        solve(ref, def);
        ref.detach_spans();
        b.detach_spans();
        const SolverBatch& cb = b;
        const SolverBatch& cr2 = ref;
        for (Index i = 0; i < 4; ++i) {
            CHECK(cb.state_at(i, 0) == cr2.state_at(i, 0));
            CHECK(cb.state_at(i, 1) == cr2.state_at(i, 1));
        }
        CHECK(cb.state_at(2, 0) == cb.state_at(2, 0) && cb.outcomes()[2].accepted_steps > 10);
    });

    run_case("detection observer (solve.hpp:46-50) through the device log", [] {
        // valve: impacts (event 1, restitution action) until the stop event
        const Index n = 64;
        ProblemPool pool(PoolDims{n, 3, 5, 2});
        for (Index i = 0; i < n; ++i) {
            pool.time_start(i) = 0.0;
            pool.time_end(i) = 1e6;
            const Real q = 0.2 + 9.8 * static_cast<Real>(i) / static_cast<Real>(n - 1);
            const Real p[5] = {1.25, 10.0, 20.0, q, 0.8};
            for (Index c = 0; c < 5; ++c) pool.param_at(i, c) = p[c];
            pool.state_at(i, 0) = 0.2;
            pool.state_at(i, 1) = 0.0;
            pool.state_at(i, 2) = 10.2;
        }
        models::ValveSystem def;
        SolverBatch b(make_batch_dims(n, def.dims()));
        linear_set(b, pool, {0, 0, n, CopyMode::All});
        std::vector<Index> per_system(static_cast<std::size_t>(n), 0);
        Index impacts = 0, last_sys = -1, bad_order = 0, bad_action = 0;
        auto on_det = [&](Index s, const Detection& d, std::span<const Real> pre, std::span<const Real> post) {
            if (s < last_sys) ++bad_order;
            last_sys = s;
            ++per_system[static_cast<std::size_t>(s)];
            if (d.event_index == 1) {
                ++impacts;
                if (!(post[0] == 0.0 && post[1] == -0.8 * pre[1])) ++bad_action; // valve.hpp:66-76
            }
            if (d.counter < 1) ++bad_order;
        };
        solve(b, def, SolverConfig{Algorithm::RKCK45, 1e-3}, SolveObservers<NoBatchStepObserver, decltype(on_det)>{{}, on_det});
        const SolverBatch& cb = b;
        for (Index i = 0; i < n; ++i)
            CHECK(per_system[static_cast<std::size_t>(i)] == cb.outcomes()[static_cast<std::size_t>(i)].event_detections);
        CHECK(impacts > 0 && bad_order == 0 && bad_action == 0);
        // the same solve without an observer gives bitwise the same results
        SolverBatch plain(make_batch_dims(n, def.dims()));
        linear_set(plain, pool, {0, 0, n, CopyMode::All});
        solve(plain, def, SolverConfig{Algorithm::RKCK45, 1e-3});
        const SolverBatch& cp = plain;
        for (Index i = 0; i < 3 * n; ++i) CHECK(cp.state()[static_cast<std::size_t>(i)] == cb.state()[static_cast<std::size_t>(i)]);
    });

    run_case("random_set permutation identity", [] { // test_batch.cpp:114-139
        const Index n = 64;
        const auto pool = duffing_pool(n);
        models::DuffingSystem def;
        SolverBatch plain(make_batch_dims(n, def.dims()));
        linear_set(plain, pool, {0, 0, n, CopyMode::All});
        solve(plain, def);
        std::vector<Index> perm(n), slots(n);
        for (Index i = 0; i < n; ++i) {
            perm[static_cast<std::size_t>(i)] = (i * 37 + 11) % n;
            slots[static_cast<std::size_t>(i)] = i;
        }
        SolverBatch permuted(make_batch_dims(n, def.dims()));
        random_set(permuted, pool, {slots, perm, CopyMode::All});
        solve(permuted, def);
        const SolverBatch &cp = permuted, &cq = plain;
        for (Index i = 0; i < n; ++i) {
            CHECK(cp.state_at(i, 0) == cq.state_at(perm[static_cast<std::size_t>(i)], 0));
            CHECK(cp.state_at(i, 1) == cq.state_at(perm[static_cast<std::size_t>(i)], 1));
        }
        CHECK_THROWS_AS(random_set(permuted, pool, {{1, 1}, {0, 1}, CopyMode::All}), std::invalid_argument);
        CHECK_THROWS_AS(random_set(permuted, pool, {{64}, {0}, CopyMode::All}), std::out_of_range);
    });

    run_case("failure isolation and sticky abort", [] { // test_batch.cpp:139-167
        const Index n = 32;
        const auto pool = duffing_pool(n);
        models::DuffingSystem def;
        SolverBatch clean(make_batch_dims(n, def.dims()));
        linear_set(clean, pool, {0, 0, n, CopyMode::All});
        solve(clean, def);
        ProblemPool poisoned = pool;
        poisoned.param_at(7, 1) = std::numeric_limits<Real>::quiet_NaN();
        SolverBatch dirty(make_batch_dims(n, def.dims()));
        linear_set(dirty, poisoned, {0, 0, n, CopyMode::All});
        solve(dirty, def);
        const SolverBatch &cd = dirty, &cc = clean;
        CHECK(cd.outcomes()[7].reason == StopReason::NonFiniteAbort);
        for (Index i = 0; i < n; ++i) {
            if (i == 7) continue;
            CHECK(cd.state_at(i, 0) == cc.state_at(i, 0));
            CHECK(cd.outcomes()[static_cast<std::size_t>(i)].reason == StopReason::ReachedEndTime);
        }
        solve(dirty, def);
        CHECK(cd.outcomes()[7].reason == StopReason::NonFiniteAbort);
        linear_set(dirty, pool, {7, 7, 1, CopyMode::All});
        CHECK(cd.outcomes()[7].reason == StopReason::ReachedEndTime);
    });

    run_case("solve rejects inconsistent setups", [] { // test_batch.cpp:184-204
        const auto pool = duffing_pool(4);
        models::DuffingSystem def;
        SolverBatch batch(make_batch_dims(4, def.dims()));
        linear_set(batch, pool, {0, 0, 4, CopyMode::All});
        SolverConfig bad_step;
        bad_step.initial_time_step = 0.0;
        CHECK_THROWS_AS(solve(batch, def, bad_step), std::invalid_argument);
        SolverConfig over_max;
        over_max.initial_time_step = 1e7;
        CHECK_THROWS_AS(solve(batch, def, over_max), std::invalid_argument);
        SolverBatch wrong(BatchDims{4, 3, 4, 0, 0});
        CHECK_THROWS_AS(solve(wrong, def), std::invalid_argument);
        auto backwards = duffing_pool(4);
        backwards.time_end(1) = -1.0;
        SolverBatch btw(make_batch_dims(4, def.dims()));
        linear_set(btw, backwards, {0, 0, 4, CopyMode::All});
        bool msg_ok = false;
        try {
            solve(btw, def);
        } catch (const std::invalid_argument& e) {
            msg_ok = std::string(e.what()) == "solve: system 1 has t1 < t0";
        }
        CHECK(msg_ok);
    });

    run_case("iterated poincare sampling feeds endpoints forward", [] { // test_driver.cpp:209-234
        models::DuffingSystem def;
        const auto pool = duffing_pool(1, 0.215);
        SolverBatch batch(make_batch_dims(1, def.dims()));
        linear_set(batch, pool, {0, 0, 1, CopyMode::All});
        const Index transient = 1024, saved = 32;
        std::vector<Real> points;
        solve_iteratively(batch, def, SolverConfig{}, transient + saved, [&](Index iter, const SolverBatch& b) {
            if (iter >= transient) points.push_back(b.state_at(0, 0));
        });
        CHECK(static_cast<Index>(points.size()) == saved);
        std::vector<Real> centers;
        for (Real v : points) {
            bool known = false;
            for (Real c : centers) known = known || std::abs(v - c) <= 1e-6;
            if (!known) centers.push_back(v);
        }
        CHECK(centers.size() <= 4);
    });

    run_case("duffing event stop lands on a local maximum", [] { // test_driver.cpp:96-108
        models::DuffingMaxEventSystem def(1e-6, 1);
        ProblemPool pool(PoolDims{1, 2, 4, 2});
        pool.time_end(0) = 1e6;
        pool.state_at(0, 0) = 0.3;
        pool.state_at(0, 1) = 0.7;
        models::DuffingParams{}.write(pool.parameters());
        SolverBatch b(make_batch_dims(1, def.dims()));
        linear_set(b, pool, {0, 0, 1, CopyMode::All});
        solve(b, def);
        const SolverBatch& cb = b;
        CHECK(cb.outcomes()[0].reason == StopReason::EventStop);
        CHECK(std::abs(cb.state_at(0, 1)) <= 1e-6);
        CHECK(cb.accessory_at(0, 0) == cb.state_at(0, 0));
    });

    run_case("fetch order changes no result (set_fetch_order)", [] {
        models::DuffingMaxEventSystem def(1e-6, 0);
        const Index n = 3000;
        ProblemPool pool(PoolDims{n, 2, 4, 2});
        for (Index i = 0; i < n; ++i) {
            pool.time_end(i) = 2.0 * std::numbers::pi;
            pool.param_at(i, 0) = 0.2 + 0.1 * Real(i % 50) / 49.0; // k
            pool.param_at(i, 1) = 0.1 + 0.4 * Real(i / 50) / 59.0;  // B
            pool.param_at(i, 2) = 1.0;                                // delta
            pool.param_at(i, 3) = 1.0;                                // omega
        }
        SolverBatch a(make_batch_dims(n, def.dims())), b(make_batch_dims(n, def.dims()));
        a.set_fetch_order(ODEGPU_FETCH_NATURAL);
        b.set_fetch_order(ODEGPU_FETCH_COST);
        linear_set(a, pool, {0, 0, n, CopyMode::All});
        linear_set(b, pool, {0, 0, n, CopyMode::All});
        solve_iteratively(a, def, SolverConfig{}, 3, [](Index, const SolverBatch&) {});
        solve_iteratively(b, def, SolverConfig{}, 3, [](Index, const SolverBatch&) {});
        const SolverBatch &ca = a, &cb = b;
        bool same = true;
        for (Index i = 0; i < n; ++i)
            same = same && ca.state_at(i, 0) == cb.state_at(i, 0) && ca.state_at(i, 1) == cb.state_at(i, 1) &&
                   ca.accessory_at(i, 0) == cb.accessory_at(i, 0) &&
                   ca.outcomes()[std::size_t(i)].rejected_steps == cb.outcomes()[std::size_t(i)].rejected_steps;
        CHECK(same);
        CHECK_THROWS_AS(a.set_fetch_order(9), std::invalid_argument);
    });

    run_case("bubble scan smoke: every iteration stops at a located maximum", [] { // test_scan.cpp:176-196
        // 1 (pa1) x 1 (pa2) x 2 (f1) x 3 (f2) grid, 8 transient + 4 saved iterations
        const std::vector<Real> f1 = {20.0, 1000.0}, f2 = {20.0, 141.42135623730951, 1000.0};
        ProblemPool pool(PoolDims{6, 2, 13, 4});
        Index i = 0;
        for (Real a : f1)
            for (Real b : f2) {
                models::BubblePhysical phys;
                phys.pa1 = 1.1e5;
                phys.pa2 = 0.0;
                phys.omega1 = a * 1e3 * kTwoPi;
                phys.omega2 = b * 1e3 * kTwoPi;
                models::bubble_coefficients(phys).write(
                    std::span<Real>(std::vector<Real>(13).data(), 13)); // API parity
                const auto c = models::bubble_coefficients(phys);
                for (Index k = 0; k < 13; ++k) pool.param_at(i, k) = c[static_cast<std::size_t>(k)];
                pool.time_end(i) = 1e6;
                pool.state_at(i, 0) = 1.0;
                ++i;
            }
        models::BubbleCollapseSystem def(1e-6);
        SolverBatch b(make_batch_dims(6, def.dims()));
        linear_set(b, pool, {0, 0, 6, CopyMode::All});
        Index event_stops = 0;
        std::vector<Real> prev_t0(6, 0.0);
        bool increasing = true;
        SolverConfig cfg;
        solve_iteratively(b, def, cfg, 12, [&](Index, const SolverBatch& bb) {
            for (Index s = 0; s < 6; ++s) {
                event_stops += bb.outcomes()[static_cast<std::size_t>(s)].reason == StopReason::EventStop;
                increasing = increasing && bb.time_start(s) > prev_t0[static_cast<std::size_t>(s)];
                prev_t0[static_cast<std::size_t>(s)] = bb.time_start(s);
            }
        });
        CHECK(event_stops == 6 * 12);
        CHECK(increasing);
    });

    run_case("valve impacts at low flow rate, equilibrium at high", [] { // test_scan.cpp:198-219
        models::ValveSystem def(1e-6);
        auto run = [&](Real q, Index transient, Index saved, std::vector<std::pair<Real, Real>>& rows,
                       Index& equilibria) {
            ProblemPool pool(PoolDims{1, 3, 5, 2});
            models::ValveParams{1.25, 10.0, 20.0, q, 0.8}.write(pool.parameters());
            pool.time_end(0) = 1e6;
            pool.state_at(0, 0) = 0.2;
            pool.state_at(0, 2) = 10.2;
            SolverBatch b(make_batch_dims(1, def.dims()));
            linear_set(b, pool, {0, 0, 1, CopyMode::All});
            solve_iteratively(b, def, SolverConfig{}, transient + saved, [&](Index it, const SolverBatch& bb) {
                equilibria += bb.outcomes()[0].reason == StopReason::EquilibriumStop;
                if (it >= transient) rows.emplace_back(bb.accessory_at(0, 0), bb.accessory_at(0, 1));
            });
        };
        std::vector<std::pair<Real, Real>> rows;
        Index eq = 0;
        run(1.0, 24, 4, rows, eq);
        CHECK(rows.size() == 4);
        for (auto [mx, mn] : rows) {
            CHECK(std::abs(mn) <= 1e-6);
            CHECK(mx > 0.1);
        }
        rows.clear();
        eq = 0;
        run(9.0, 256, 8, rows, eq);
        CHECK(std::abs(rows.back().first - rows.back().second) < 1e-3);
        CHECK(eq > 0);
    });

    run_case("lyapunov separates periodic from chaotic damping", [] { // test_scan.cpp:162-174
        models::DuffingLyapunovSystem def;
        ProblemPool pool(PoolDims{2, 4, 4, 1});
        const Real ks[2] = {0.215, 0.24}; // periodic window, chaotic band
        for (Index i = 0; i < 2; ++i) {
            pool.time_end(i) = kTwoPi;
            pool.state_at(i, 2) = 1.0;
            models::DuffingParams p{ks[i], 0.3, 1.0, 1.0};
            pool.param_at(i, 0) = p.k;
            pool.param_at(i, 1) = p.B;
            pool.param_at(i, 2) = p.delta;
            pool.param_at(i, 3) = p.omega;
        }
        SolverBatch b(make_batch_dims(2, def.dims()));
        linear_set(b, pool, {0, 0, 2, CopyMode::All});
        std::vector<std::vector<Real>> samples(2);
        solve_iteratively(b, def, SolverConfig{}, 256 + 64, [&](Index it, const SolverBatch& bb) {
            if (it < 256) return;
            for (Index s = 0; s < 2; ++s) samples[static_cast<std::size_t>(s)].push_back(bb.accessory_at(s, 0));
            CHECK(bb.state_at(0, 2) == 1.0); // radius reset by finalize
        });
        CHECK(models::lyapunov_accumulate(samples[0], kTwoPi) < 0.0);
        CHECK(models::lyapunov_accumulate(samples[1], kTwoPi) > 0.0);
    });

    run_case("validate_definition (test_system.cpp:42-81)", [] {
        models::DuffingSystem duffing;
        const Real y0[] = {0.0, 0.0};
        const Real p0[] = {0.2, 0.3, 1.0, 1.0};
        validate_definition(duffing, 0.0, std::span<const Real>(y0), std::span<const Real>(p0));
        models::ValveSystem valve;
        const Real yv[] = {0.2, 0.0, 10.2};
        const Real pv[] = {1.25, 10.0, 20.0, 0.3, 0.8};
        validate_definition(valve, 0.0, std::span<const Real>(yv), std::span<const Real>(pv));
        bool named = false;
        try {
            validate_definition(ShortEventDef{}, 0.0, std::span<const Real>(y0), {});
        } catch (const std::invalid_argument& e) {
            named = std::string(e.what()).find("event_values") != std::string::npos;
        }
        CHECK(named);
        const Real y1[] = {0.0};
        ControlsDef good;
        good.ode = OdeControls::uniform(1, 1e-9, 1e-9);
        validate_definition(good, 0.0, std::span<const Real>(y1), {});
        const auto rejected = [&](auto&& mutate) {
            ControlsDef bad;
            bad.ode = OdeControls::uniform(1, 1e-9, 1e-9);
            mutate(bad.ode);
            CHECK_THROWS_AS(validate_definition(bad, 0.0, std::span<const Real>(y1), {}), std::invalid_argument);
        };
        rejected([](OdeControls& c) { c.min_step = 2.0 * c.max_step; });
        rejected([](OdeControls& c) { c.abs_tol[0] = 0.0; });
        rejected([](OdeControls& c) { c.rel_tol[0] = std::numeric_limits<Real>::quiet_NaN(); });
        rejected([](OdeControls& c) { c.step_grow_limit = 1.0; });
        rejected([](OdeControls& c) { c.step_shrink_limit = 1.5; });
        rejected([](OdeControls& c) { c.rel_tol.push_back(1e-9); });
    });

    run_case("scan protocols: rows, order, diagnostics, CSV (scan.hpp)", [] { // test_scan.cpp:49-131
        scan::DuffingScanSpec spec;
        spec.k = scan::ParamRange{0.2, 0.3, 24, scan::Scale::Linear};
        spec.transient = 3;
        spec.saved = 2;
        spec.solver.batch_capacity = 10; // 3 chunks
        const auto acc = scan::run_duffing_maxima(spec, scan::MaximaMode::Accessory);
        CHECK(acc.columns == std::vector<std::string>({"k", "y1_max", "status"}));
        CHECK(acc.rows.size() == 48);
        CHECK(acc.rows[0][0] == 0.2 && acc.rows[9][0] == spec.k.values()[9]); // chunk-major, iteration, system
        CHECK(acc.diagnostics.reason_counts[0] == 24 * 5);
        // test_scan.cpp:132-159: on a converged periodic window both
        // recordings agree on the envelope over the saved iterations
        scan::DuffingScanSpec w;
        w.k = scan::ParamRange{0.21, 0.22, 3, scan::Scale::Linear};
        w.transient = 512;
        w.saved = 4;
        const auto wa = scan::run_duffing_maxima(w, scan::MaximaMode::Accessory);
        const auto ev = scan::run_duffing_maxima(w, scan::MaximaMode::Event);
        CHECK(wa.rows.size() == 12 && ev.rows.size() == 12);
        CHECK(wa.diagnostics.detections == 0);
        CHECK(ev.diagnostics.detections > 0);
        CHECK(ev.diagnostics.detections_outside_zone == 0);
        CHECK(ev.diagnostics.max_residual_ratio > 0 && ev.diagnostics.max_residual_ratio <= 1.0);
        for (std::size_t k = 0; k < 3; ++k) {
            Real env_acc = -1e300, env_evt = -1e300;
            for (std::size_t i = 0; i < 4; ++i) {
                env_acc = std::max(env_acc, wa.rows[3 * i + k][1]);
                env_evt = std::max(env_evt, ev.rows[3 * i + k][1]);
            }
            // doctest::Approx(env_evt).epsilon(1e-4): eps * (scale 1 + max magnitude)
            CHECK(std::abs(env_acc - env_evt) < 1e-4 * (1.0 + std::max(std::abs(env_acc), std::abs(env_evt))));
        }
        scan::BubbleScanSpec b;
        b.f1_khz = scan::ParamRange{20.0, 1000.0, 3, scan::Scale::Log};
        b.f2_khz = scan::ParamRange{20.0, 1000.0, 3, scan::Scale::Log};
        b.transient = 4;
        b.saved = 4;
        const auto br = scan::run_bubble_scan(b);
        CHECK(br.rows.size() == 9);
        CHECK(br.diagnostics.reason_counts[1] == 72); // test_scan.cpp:195
        CHECK(br.diagnostics.start_times_strictly_increase);
        const std::string path = "/tmp/odegpu_scan_test.csv";
        scan::emit_rows(path, acc.columns, acc.rows);
        std::FILE* f = std::fopen(path.c_str(), "r");
        CHECK(f != nullptr);
        char line[256];
        CHECK(std::fgets(line, sizeof line, f) && std::string(line) == "# k,y1_max,status\n");
        double k = 0, y = 0, st = 0;
        CHECK(std::fscanf(f, "%lf,%lf,%lf", &k, &y, &st) == 3 && k == acc.rows[0][0] && y == acc.rows[0][1]);
        std::fclose(f);
        bool threw = false;
        try {
            scan::ParamRange{0.0, 1.0, 4, scan::Scale::Log}.values();
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        CHECK(threw);
    });

    std::printf("%d checks, %d failed\n", g_checks, g_failed);
    return g_failed;
}
