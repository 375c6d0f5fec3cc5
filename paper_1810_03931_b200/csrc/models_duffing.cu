// models_duffing.cu — solve-kernel instantiations of the Duffing models
// (models/duffing.hpp; DuffingMaxMin is the cfg1 harness model).
#include "launch.cuh"
#include "odegpu/models/duffing.hpp"

namespace odegpu::device {
template <>
struct KernelPolicy<odegpu::models::DuffingMaxMinHooks> {
    static constexpr bool kRolledStages = false, kColdInShared = false, kParamsInShared = false;
};
} // namespace odegpu::device

namespace odegpu::detail {

// Policies from the variant sweep (profiles/r01_variants.md):
// * cfg1 (RK4 + max/min accessories, only 46 080 systems = 2.4 blocks/SM):
//   occupancy is not the limit, so all state stays in registers (0.615 ms vs
//   0.72 ms with the cold state in shared memory).
// * the event / accessory RKCK45 models: cold state in shared memory frees
//   enough registers (123 -> 72) for 7 blocks of 128 threads per SM.
// * adaptive models take up systems longest first (kCostOrder, DESIGN.md
//   §3.1): cfg2 2.09 -> 1.92 ms.
template <>
struct LaunchPolicy<models::DuffingMaxMinHooks> {
#ifdef ODEGPU_CFG1_BLOCK
    static constexpr int kBlock = ODEGPU_CFG1_BLOCK;
#endif
    static constexpr int kMinBlocks = ODEGPU_MB(1);
};
template <>
struct LaunchPolicy<models::DuffingMaxEventHooks> {
    static constexpr int kMinBlocks = ODEGPU_MB(6);
    static constexpr bool kCostOrder = true;
};
template <>
struct LaunchPolicy<models::DuffingMaxAccessoryHooks> {
    static constexpr int kMinBlocks = ODEGPU_MB(6);
    static constexpr bool kCostOrder = true;
};
template <>
struct LaunchPolicy<models::DuffingHooks> {
    static constexpr int kMinBlocks = ODEGPU_MB(6);
    static constexpr bool kCostOrder = true;
};
// 4-dim Lyapunov system: 3 blocks/SM (<= 168 regs) keeps it spill-free.
template <>
struct LaunchPolicy<models::DuffingLyapunovHooks> {
    static constexpr int kMinBlocks = ODEGPU_MB(3);
    static constexpr bool kCostOrder = true;
};

bool family_dims_duffing(const odegpu_model& m, odegpu_system_dims* d, bool* keeps, bool* fusable) {
    switch (m.id) {
    case ODEGPU_MODEL_DUFFING: set_dims<models::DuffingHooks>(d, keeps, fusable); return true;
    case ODEGPU_MODEL_DUFFING_MAX_ACCESSORY: set_dims<models::DuffingMaxAccessoryHooks>(d, keeps, fusable); return true;
    case ODEGPU_MODEL_DUFFING_MAX_EVENT: set_dims<models::DuffingMaxEventHooks>(d, keeps, fusable); return true;
    case ODEGPU_MODEL_DUFFING_MAXMIN: set_dims<models::DuffingMaxMinHooks>(d, keeps, fusable); return true;
    case ODEGPU_MODEL_DUFFING_LYAPUNOV: set_dims<models::DuffingLyapunovHooks>(d, keeps, fusable); return true;
    default: return false;
    }
}

bool family_launch_duffing(odegpu_batch* b, const odegpu_model& m, int alg, const dev::Controls& c) {
    switch (m.id) {
    case ODEGPU_MODEL_DUFFING: launch_alg(b, models::DuffingHooks{}, alg, c); return true;
    case ODEGPU_MODEL_DUFFING_MAX_ACCESSORY: launch_alg(b, models::DuffingMaxAccessoryHooks{}, alg, c); return true;
    case ODEGPU_MODEL_DUFFING_MAX_EVENT: launch_alg(b, models::DuffingMaxEventHooks{}, alg, c); return true;
    case ODEGPU_MODEL_DUFFING_MAXMIN: launch_alg(b, models::DuffingMaxMinHooks{}, alg, c); return true;
    case ODEGPU_MODEL_DUFFING_LYAPUNOV: launch_alg(b, models::DuffingLyapunovHooks{}, alg, c); return true;
    default: return false;
    }
}

} // namespace odegpu::detail
