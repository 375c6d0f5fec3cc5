// models_duffing.cu — solve-kernel instantiations of the Duffing models
// (models/duffing.hpp; DuffingMaxMin is the cfg1 harness model).
#include "launch.cuh"
#include "odegpu/models/duffing.hpp"

namespace odegpu::detail {

// 4-dim Lyapunov system: 156 registers unbounded; 3 blocks/SM (<= 168 regs) keeps it spill-free.
template <>
struct LaunchPolicy<models::DuffingLyapunovHooks> {
    static constexpr int kMinBlocks = 3;
};

bool family_dims_duffing(const odegpu_model& m, odegpu_system_dims* d) {
    switch (m.id) {
    case ODEGPU_MODEL_DUFFING: set_dims<models::DuffingHooks>(d); return true;
    case ODEGPU_MODEL_DUFFING_MAX_ACCESSORY: set_dims<models::DuffingMaxAccessoryHooks>(d); return true;
    case ODEGPU_MODEL_DUFFING_MAX_EVENT: set_dims<models::DuffingMaxEventHooks>(d); return true;
    case ODEGPU_MODEL_DUFFING_MAXMIN: set_dims<models::DuffingMaxMinHooks>(d); return true;
    case ODEGPU_MODEL_DUFFING_LYAPUNOV: set_dims<models::DuffingLyapunovHooks>(d); return true;
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
