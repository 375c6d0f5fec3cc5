// models_keller_miksis.cu — solve-kernel instantiations of the bubble models
// (models/keller_miksis.hpp).
#include "launch.cuh"
#include "odegpu/models/keller_miksis.hpp"

// Keller-Miksis: the RHS (pow + 2 sincos + 4 quotients) is large. It is an
// outlined call (one copy of its code, its own register allocation), so the
// six stages can be straight-line with k1..k6 in registers — no stage switch,
// no shared-memory stage vectors: 96 registers instead of the 128 the inlined
// rolled loop needed. With the bookkeeping in registers and the cold state +
// 13 coefficients in shared memory (40 KB per block) 5 blocks of 128 fit per
// SM: 15.5 -> 14.4 ms on cfg3 (rolled/inlined, 4 blocks) — DESIGN.md §3.1.
// The time-term cache keeps one slot (the step's end point, 3 KB per block):
// 5 blocks still fit, 13.0 -> 12.6 ms; with two slots the fifth block is
// lost (15.1 ms).
namespace odegpu::device {
template <>
struct KernelPolicy<odegpu::models::BubbleCollapseHooks> {
    static constexpr bool kRolledStages = false, kColdInShared = true, kParamsInShared = true, kBookInShared = false,
                          kOutlineRhs = true;
};
template <>
struct KernelPolicy<odegpu::models::KellerMiksisHooks> {
    static constexpr bool kRolledStages = false, kColdInShared = true, kParamsInShared = true, kBookInShared = false,
                          kOutlineRhs = true;
};
} // namespace odegpu::device

namespace odegpu::detail {

// Keller-Miksis systems are taken up in index order under AUTO. Longest
// first by the previous iteration (the cost order) measured even at 2^24
// (bench cfg5: 10.96 vs 10.96 G steps/s) and 2 % behind at 2^20 (cfg3: 9.49
// vs 9.67; profiles/r02ai/), and it scatters a warp's entry / exit accesses
// over 32 distant systems: 10.1 GB of DRAM traffic per in-place iteration
// of the 2^24 pool against 4.7 GB algorithmic (ncu, profiles/r02ag_ncu_summary.md).
// With ~226 systems per lane at 2^24 and the fused iterations, the end-of-
// pool tail the order was for is no longer there. -DODEGPU_KM_COST_ORDER=true
// restores it (tuning).
#ifndef ODEGPU_KM_COST_ORDER
#define ODEGPU_KM_COST_ORDER false
#endif

template <>
struct LaunchPolicy<models::BubbleCollapseHooks> {
    static constexpr int kMinBlocks = ODEGPU_MB(5);
    static constexpr bool kCostOrder = ODEGPU_KM_COST_ORDER;
};
template <>
struct LaunchPolicy<models::KellerMiksisHooks> {
    static constexpr int kMinBlocks = ODEGPU_MB(5);
    static constexpr bool kCostOrder = ODEGPU_KM_COST_ORDER;
};

// 5 resident blocks need 5 x (layout + 1 KB reserved) <= 228 KB of shared
// memory per SM: every byte of per-lane cold state counts (solver.cuh
// ColdState packs its flags and secant indices into bytes for this).
static_assert(5 * (dev::solve_smem_bytes<models::BubbleCollapseHooks, Algorithm::RKCK45, kBlock>() + 1024) <=
                  228 * 1024,
              "Keller-Miksis shared-memory layout no longer fits 5 blocks per SM");

bool family_dims_keller_miksis(const odegpu_model& m, odegpu_system_dims* d, bool* keeps, bool* fusable) {
    switch (m.id) {
    case ODEGPU_MODEL_KELLER_MIKSIS: set_dims<models::KellerMiksisHooks>(d, keeps, fusable); return true;
    case ODEGPU_MODEL_BUBBLE_COLLAPSE: set_dims<models::BubbleCollapseHooks>(d, keeps, fusable); return true;
    default: return false;
    }
}

bool family_launch_keller_miksis(odegpu_batch* b, const odegpu_model& m, int alg, const dev::Controls& c) {
    switch (m.id) {
    case ODEGPU_MODEL_KELLER_MIKSIS: launch_alg(b, models::KellerMiksisHooks{}, alg, c); return true;
    case ODEGPU_MODEL_BUBBLE_COLLAPSE: launch_alg(b, models::BubbleCollapseHooks{}, alg, c); return true;
    default: return false;
    }
}

} // namespace odegpu::detail
