// models_keller_miksis.cu — solve-kernel instantiations of the bubble models
// (models/keller_miksis.hpp).
#include "launch.cuh"
#include "odegpu/models/keller_miksis.hpp"

namespace odegpu::detail {

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
