// Host check of the TimeSplitHooks contract (include/odegpu/hooks.hpp): for
// every built-in time-split model, ode_rhs(t, y, p) equals time_terms(t, p)
// followed by ode_rhs_split bit for bit, on seeded random inputs. (The device
// side is checked end to end: scripts/compare_libs.py.)
#include <cstdio>
#include <cstring>
#include <random>

#include "odegpu/models/duffing.hpp"
#include "odegpu/models/keller_miksis.hpp"

using namespace odegpu;

template <class H>
static int check(const char* name, std::mt19937_64& rng, double tmax) {
    static_assert(TimeSplitHooks<H>);
    constexpr int N = H::kSystemDim, P = H::kParamCount, K = H::kTimeTermCount;
    std::uniform_real_distribution<double> u(-1.0, 1.0), pos(0.05, 3.0), tt(-tmax, tmax);
    int bad = 0;
    for (int trial = 0; trial < 20000; ++trial) {
        double y[N], p[P], a[N], b[N], terms[K];
        for (double& v : y) v = (trial & 1) ? pos(rng) : u(rng);
        for (double& v : p) v = pos(rng);
        const double t = tt(rng);
        H h{};
        h.ode_rhs(t, y, p, a);
        h.time_terms(t, p, terms);
        h.ode_rhs_split(t, y, p, terms, b);
        if (std::memcmp(a, b, sizeof a) != 0) ++bad;
    }
    std::printf("%s: %d mismatches\n", name, bad);
    return bad;
}

int main() {
    std::mt19937_64 rng(123);
    int bad = check<models::DuffingMaxEventHooks>("duffing", rng, 100.0);
    bad += check<models::DuffingMaxMinHooks>("duffing_maxmin", rng, 100.0);
    bad += check<models::BubbleCollapseHooks>("keller_miksis", rng, 100.0);
    static_assert(!TimeSplitHooks<models::DuffingLyapunovHooks>);
    return bad == 0 ? 0 : 1;
}
