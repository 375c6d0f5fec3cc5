// models_fakes.cu — solve-kernel instantiations of the reference test-suite
// fakes (test_fakes.cuh), so its known answers run through the product path.
#include "launch.cuh"
#include "test_fakes.cuh"

// Two of the fakes run the kernel structures no built-in model uses any
// more, so the golden tests keep them covered: the rolled stage loop with
// shared-memory stage vectors (SeatContact: 3 states, 2 events, impact) and
// the outlined RHS with the bookkeeping in shared memory (Ramp: secant,
// stops, direction filter).
namespace odegpu::device {
template <>
struct KernelPolicy<fakes::SeatContactHooks> {
    static constexpr bool kRolledStages = true, kColdInShared = true, kParamsInShared = true, kBookInShared = true;
};
template <>
struct KernelPolicy<fakes::RampHooks> {
    static constexpr bool kRolledStages = false, kColdInShared = true, kParamsInShared = false, kBookInShared = true,
                          kOutlineRhs = true;
};
} // namespace odegpu::device

namespace odegpu::detail {

bool family_dims_fakes(const odegpu_model& m, odegpu_system_dims* d, bool* keeps, bool* fusable) {
    switch (m.id) {
    case ODEGPU_MODEL_CONSTANT: set_dims<fakes::ConstantHooks>(d, keeps, fusable); return true;
    case ODEGPU_MODEL_CUBIC_TIME: set_dims<fakes::CubicTimeHooks>(d, keeps, fusable); return true;
    case ODEGPU_MODEL_EXPONENTIAL: set_dims<fakes::ExponentialHooks>(d, keeps, fusable); return true;
    case ODEGPU_MODEL_UNIT_SLOPE: set_dims<fakes::UnitSlopeHooks>(d, keeps, fusable); return true;
    case ODEGPU_MODEL_COUNTING: set_dims<fakes::CountingHooks>(d, keeps, fusable); return true;
    case ODEGPU_MODEL_RAMP: set_dims<fakes::RampHooks>(d, keeps, fusable); return true;
    case ODEGPU_MODEL_DECAY: set_dims<fakes::DecayHooks>(d, keeps, fusable); return true;
    case ODEGPU_MODEL_SEAT_CONTACT: set_dims<fakes::SeatContactHooks>(d, keeps, fusable); return true;
    case ODEGPU_MODEL_HARMONIC: set_dims<fakes::HarmonicHooks>(d, keeps, fusable); return true;
    case ODEGPU_MODEL_BLOWUP: set_dims<fakes::BlowUpHooks>(d, keeps, fusable); return true;
    default: return false;
    }
}

bool family_launch_fakes(odegpu_batch* b, const odegpu_model& m, int alg, const dev::Controls& c) {
    const double* k = m.consts;
    switch (m.id) {
    case ODEGPU_MODEL_CONSTANT: {
        fakes::ConstantHooks h;
        h.value = k[0];
        launch_alg(b, h, alg, c);
        return true;
    }
    case ODEGPU_MODEL_CUBIC_TIME: launch_alg(b, fakes::CubicTimeHooks{}, alg, c); return true;
    case ODEGPU_MODEL_EXPONENTIAL: launch_alg(b, fakes::ExponentialHooks{}, alg, c); return true;
    case ODEGPU_MODEL_UNIT_SLOPE: launch_alg(b, fakes::UnitSlopeHooks{}, alg, c); return true;
    case ODEGPU_MODEL_COUNTING: launch_alg(b, fakes::CountingHooks{}, alg, c); return true;
    case ODEGPU_MODEL_RAMP: {
        fakes::RampHooks h;
        h.slope = k[0];
        h.level = k[1];
        launch_alg(b, h, alg, c);
        return true;
    }
    case ODEGPU_MODEL_DECAY: launch_alg(b, fakes::DecayHooks{}, alg, c); return true;
    case ODEGPU_MODEL_SEAT_CONTACT: launch_alg(b, fakes::SeatContactHooks{}, alg, c); return true;
    case ODEGPU_MODEL_HARMONIC: launch_alg(b, fakes::HarmonicHooks{}, alg, c); return true;
    case ODEGPU_MODEL_BLOWUP: launch_alg(b, fakes::BlowUpHooks{}, alg, c); return true;
    default: return false;
    }
}

} // namespace odegpu::detail
