// models_valve.cu — solve-kernel instantiation of the impacting valve
// (models/valve.hpp).
#include "launch.cuh"
#include "odegpu/models/valve.hpp"

namespace odegpu::detail {

bool family_dims_valve(const odegpu_model& m, odegpu_system_dims* d) {
    if (m.id != ODEGPU_MODEL_VALVE) return false;
    set_dims<models::ValveHooks>(d);
    return true;
}

bool family_launch_valve(odegpu_batch* b, const odegpu_model& m, int alg, const dev::Controls& c) {
    if (m.id != ODEGPU_MODEL_VALVE) return false;
    launch_alg(b, models::ValveHooks{}, alg, c);
    return true;
}

} // namespace odegpu::detail
