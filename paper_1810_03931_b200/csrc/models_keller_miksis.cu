// models_keller_miksis.cu — solve-kernel instantiations of the bubble models
// (models/keller_miksis.hpp).
#include "launch.cuh"
#include "odegpu/models/keller_miksis.hpp"

namespace odegpu::device {
template <>
struct KernelPolicy<odegpu::models::BubbleCollapseHooks> {
    static constexpr bool kRolledStages = true, kColdInShared = true, kParamsInShared = true, kBookInShared = true;
};
} // namespace odegpu::device

namespace odegpu::device {
template <>
struct KernelPolicy<odegpu::models::KellerMiksisHooks> {
    static constexpr bool kRolledStages = true, kColdInShared = true, kParamsInShared = true, kBookInShared = true;
};
} // namespace odegpu::device

namespace odegpu::detail {

// Keller-Miksis: the RHS (pow + 2 sincos + 4 divisions) is large, so the six
// stages share one RHS call site (rolled loop: I-cache) and both the cold
// state and the 13 coefficients live in shared memory (profiles/r01_variants.md:
// 22.98 ms vs 24.1 ms unrolled). 4 blocks/SM: at 5 ptxas spills 84 B, and the
// stage vectors must stay in registers.
template <>
struct LaunchPolicy<models::BubbleCollapseHooks> {
    static constexpr int kMinBlocks = ODEGPU_MB(4);
};
template <>
struct LaunchPolicy<models::KellerMiksisHooks> {
    static constexpr int kMinBlocks = ODEGPU_MB(4);
};

bool family_dims_keller_miksis(const odegpu_model& m, odegpu_system_dims* d) {
    switch (m.id) {
    case ODEGPU_MODEL_KELLER_MIKSIS: set_dims<models::KellerMiksisHooks>(d); return true;
    case ODEGPU_MODEL_BUBBLE_COLLAPSE: set_dims<models::BubbleCollapseHooks>(d); return true;
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
