// custom.cuh — solving user-defined system models (the reference's
// SystemModel plugin API, /root/reference/proj/include/odensemble/
// system.hpp:49-65) on the GPU.
//
// A user model is a host class (dims(), ode_controls(), event_controls())
// whose hooks live in a trivially copyable `hooks_type` annotated ODEGPU_HD
// (include/odegpu/hooks.hpp). Including this header in a translation unit
// compiled by nvcc makes odegpu::solve / solve_iteratively work for it: the
// solve kernel is instantiated right here, with the hooks inlined, and
// launched on the batch's device arrays through odegpu_custom_begin/_end
// (same validation and errors as the built-in models).
#ifndef ODEGPU_DEVICE_CUSTOM_CUH
#define ODEGPU_DEVICE_CUSTOM_CUH

#if !defined(__CUDACC__)
#error "odegpu/device/custom.cuh instantiates solve kernels: compile this translation unit with nvcc"
#endif

#include <cuda_runtime.h>

#include <algorithm>

#include "odegpu.h"
#include "odegpu/batch.hpp"
#include "odegpu/device/solver.cuh"
#include "odegpu/solve.hpp"

namespace odegpu {

/// Launch policy of a custom model's kernel: threads per block and the
/// __launch_bounds__ residency hint (specialise for tuning).
template <class H>
struct CustomLaunchPolicy {
    static constexpr int kBlock = 128;
    static constexpr int kMinBlocks = 4;
};

template <SystemModel D>
void solve_custom(SolverBatch& batch, const D& def, const SolverConfig& cfg) {
    using H = typename D::hooks_type;
    using LP = CustomLaunchPolicy<H>;
    detail::CControls c(def, cfg);
    const SystemDims sd = def.dims();
    const odegpu_system_dims dims{sd.system_dim, sd.param_count, sd.event_count, sd.accessory_count};
    if (sd.system_dim != H::kSystemDim || sd.param_count != H::kParamCount || sd.event_count != H::kEventCount ||
        sd.accessory_count != H::kAccessoryCount)
        throw std::invalid_argument("solve: definition dims() disagree with its hooks' widths");
    batch.push();
    odegpu_device_view v{};
    detail::check(odegpu_custom_begin(batch.handle(), &dims, &c.c_cfg, &c.c_ode, &c.c_ev, &v));
    const device::Controls ctl = device::controls_from(dims, c.c_cfg, c.c_ode, &c.c_ev);
    const device::BatchArrays a{v.time_domain, v.state, v.parameters, v.accessories, v.final_t,
                                v.reason, v.accepted_steps, v.rejected_steps, v.event_detections,
                                v.secant_failures, v.smallest_step, v.capacity, v.count, v.work};
    const H& hooks = def;
    auto launch = [&](auto kern, std::size_t smem) {
        if (smem > 48 * 1024)
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        int resident = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&resident, kern, LP::kBlock, smem);
        const Index persistent = Index(v.num_sms) * std::max(resident, 1);
        const Index needed = (v.count + LP::kBlock - 1) / LP::kBlock;
        const int grid = static_cast<int>(std::max<Index>(1, std::min(needed, persistent)));
        kern<<<grid, LP::kBlock, smem, static_cast<cudaStream_t>(v.stream)>>>(hooks, a, ctl, v.skip);
    };
    int prev = -1;
    cudaGetDevice(&prev);
    if (prev != v.device) cudaSetDevice(v.device);
    if constexpr (device::TrigCertifiable<H>) { // see include/odegpu/trig.hpp
        auto* flags = const_cast<unsigned long long*>(v.skip);
        cudaMemsetAsync(flags + 1, 0, sizeof(unsigned long long), static_cast<cudaStream_t>(v.stream));
        const int g = static_cast<int>(std::max<Index>(1, std::min<Index>((v.count + 255) / 256, Index(v.num_sms) * 8)));
        device::trig_certificate_kernel<H><<<g, 256, 0, static_cast<cudaStream_t>(v.stream)>>>(a, flags);
    }
    if (cfg.algorithm == Algorithm::RK4)
        launch(device::guarded_solve_kernel<H, Algorithm::RK4, LP::kBlock, LP::kMinBlocks>,
               device::solve_smem_bytes<H, Algorithm::RK4, LP::kBlock>());
    else
        launch(device::guarded_solve_kernel<H, Algorithm::RKCK45, LP::kBlock, LP::kMinBlocks>,
               device::solve_smem_bytes<H, Algorithm::RKCK45, LP::kBlock>());
    if (prev >= 0 && prev != v.device) cudaSetDevice(prev);
    const int rc = odegpu_custom_end(batch.handle());
    batch.invalidate_host(detail::kSolveWrites);
    detail::check(rc);
}

} // namespace odegpu

#endif
