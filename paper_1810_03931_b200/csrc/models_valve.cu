// models_valve.cu — solve-kernel instantiation of the impacting valve
// (models/valve.hpp).
#include "launch.cuh"
#include "odegpu/models/valve.hpp"

namespace odegpu::device {
// per-step bookkeeping parked in shared memory: 80 registers at 6 blocks/SM
// without spills (it spills 24 B with the bookkeeping in registers)
template <>
struct KernelPolicy<odegpu::models::ValveHooks> {
    static constexpr bool kRolledStages = false, kColdInShared = true, kParamsInShared = false, kBookInShared = true;
};
} // namespace odegpu::device

namespace odegpu::detail {

// Valve: small RHS, straight-line stages, cold state in shared memory,
// 6 blocks/SM (80 registers, spill-free; profiles/r01_variants.md: 3.60 ms
// vs 4.72 ms all-register; 7 blocks spills 8 B since the constant-bank
// tableau).
template <>
struct LaunchPolicy<models::ValveHooks> {
    static constexpr int kMinBlocks = ODEGPU_MB(6);
    static constexpr bool kCostOrder = true; // step counts spread widely: longest first
};

bool family_dims_valve(const odegpu_model& m, odegpu_system_dims* d, bool* keeps, bool* fusable) {
    if (m.id != ODEGPU_MODEL_VALVE) return false;
    set_dims<models::ValveHooks>(d, keeps, fusable);
    return true;
}

bool family_launch_valve(odegpu_batch* b, const odegpu_model& m, int alg, const dev::Controls& c) {
    if (m.id != ODEGPU_MODEL_VALVE) return false;
    launch_alg(b, models::ValveHooks{}, alg, c);
    return true;
}

} // namespace odegpu::detail
