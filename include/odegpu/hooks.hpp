// hooks.hpp — the user hook contract, device side.
//
// A model is a trivially copyable struct with compile-time widths and the
// reference's hook names and std::span signatures
// (/root/reference/proj/include/odensemble/system.hpp:49-65):
//
//   ode_rhs            <- paper: OdeFunction
//   event_values       <- paper: EventFunction
//   event_action       <- paper: ActionAfterEventDetection
//   event_accessory    <- paper: EventAccessories
//   ordinary_accessory <- paper: ActionAfterSuccessfulTimeStep / OrdinaryAccessories
//   initialize         <- paper: Initialization
//   finalize           <- paper: Finalization
//
// The struct is copied by value into the kernel's parameter bank, so hook
// data (e.g. a ramp slope) costs no registers until used; the hooks are
// inlined into the per-thread step loop (never called through pointers).
// Host-only parts (ode_controls(), event_controls()) live in the System
// classes of the C++ host API (include/odegpu/system.hpp).
#ifndef ODEGPU_HOOKS_HPP
#define ODEGPU_HOOKS_HPP

#include <concepts>
#include <span>
#include <type_traits>

#include "odegpu/core.hpp"

namespace odegpu {

/// No-op implementations of every optional hook (system.hpp:70-78).
struct HookDefaults {
    ODEGPU_HD void event_values(Real, std::span<const Real>, std::span<const Real>, std::span<Real>) const {}
    ODEGPU_HD void event_action(Index, Index, Real, std::span<Real>, std::span<const Real>) const {}
    ODEGPU_HD void ordinary_accessory(Real, std::span<const Real>, std::span<const Real>, std::span<Real>) const {}
    ODEGPU_HD void event_accessory(Index, Index, Real, std::span<const Real>, std::span<const Real>,
                                   std::span<Real>) const {}
    ODEGPU_HD void initialize(Real, std::span<Real>, std::span<Real>, std::span<const Real>, std::span<Real>) const {}
    ODEGPU_HD void finalize(Real, std::span<Real>, std::span<Real>, std::span<const Real>, std::span<Real>) const {}
};

// clang-format off
/// Device-side half of the reference's SystemModel concept (system.hpp:49-65):
/// the hooks plus compile-time widths so per-thread state can live in
/// registers.
template <typename H>
concept DeviceHooks = std::is_trivially_copyable_v<H> &&
    requires(const H& d, Real t, std::span<const Real> y, std::span<const Real> p,
             std::span<Real> out, std::span<Real> my, std::span<Real> td, std::span<Real> acc,
             Index ei, Index ec) {
    { H::kSystemDim } -> std::convertible_to<Index>;
    { H::kParamCount } -> std::convertible_to<Index>;
    { H::kEventCount } -> std::convertible_to<Index>;
    { H::kAccessoryCount } -> std::convertible_to<Index>;
    { d.ode_rhs(t, y, p, out) } -> std::same_as<void>;
    { d.event_values(t, y, p, out) } -> std::same_as<void>;
    { d.event_action(ei, ec, t, my, p) } -> std::same_as<void>;
    { d.ordinary_accessory(t, y, p, acc) } -> std::same_as<void>;
    { d.event_accessory(ei, ec, t, y, p, acc) } -> std::same_as<void>;
    { d.initialize(t, td, my, p, acc) } -> std::same_as<void>;
    { d.finalize(t, td, my, p, acc) } -> std::same_as<void>;
};

/// Optional split of ode_rhs (an extension, not a reference hook): the terms
/// that depend on t and the parameters only — the excitation, cos(omega t)
/// or the driving phases' sines — and the rest. A model declaring it
/// guarantees, bit for bit,
///   ode_rhs(t, y, p, dy)  ==  { time_terms(t, p, tt); ode_rhs_split(t, y, p, tt, dy); }
/// and the solver then evaluates the time terms once per distinct stage
/// time: an accepted step's end point (stage t + h: RK4 stage 4, Cash-Karp
/// stage 5) is the next step's first stage, and a rejected step's retry
/// starts from the same t (device/solver.cuh, TimeTermCache).
template <typename H>
concept TimeSplitHooks = DeviceHooks<H> &&
    requires(const H& d, Real t, std::span<const Real> y, std::span<const Real> p, std::span<const Real> tt,
             std::span<Real> out) {
    { H::kTimeTermCount } -> std::convertible_to<Index>;
    { d.time_terms(t, p, out) } -> std::same_as<void>;
    { d.ode_rhs_split(t, y, p, tt, out) } -> std::same_as<void>;
} && (H::kTimeTermCount > 0);
// clang-format on

/// Whether consecutive solves of one system may run inside ONE kernel launch
/// (fused iterations: solve_iteratively without a sink). The reference
/// checks every system's time domain before each solve (solve.hpp:159-161)
/// and a batch's trig certificate is computed from the time domains before a
/// launch, so fusing is exact only when no iteration can leave the checked
/// time domain: finalize does not write it (the HookDefaults no-op), or the
/// model declares `static constexpr bool kFinalizeKeepsTimeDomain = true`
/// (it only moves t0 to the stop time, inside [t0, t1]).
template <class H>
inline constexpr bool kFusableIterations = [] {
    if constexpr (requires { H::kFinalizeKeepsTimeDomain; }) return bool(H::kFinalizeKeepsTimeDomain);
    else return std::is_same_v<decltype(&H::finalize), decltype(&HookDefaults::finalize)>;
}();

/// Whether a solve leaves every system's time domain exactly as it found it:
/// neither initialize nor finalize writes it (the HookDefaults no-ops), or
/// the model declares `static constexpr bool kTimeDomainUnchanged = true`
/// (hooks that override initialize / finalize without touching the time
/// domain). The chunked pipeline then does not copy time domains back to a
/// host pool they were read from (pipeline.cu).
template <class H>
inline constexpr bool kKeepsTimeDomain = [] {
    if constexpr (requires { H::kTimeDomainUnchanged; }) return bool(H::kTimeDomainUnchanged);
    else
        return std::is_same_v<decltype(&H::initialize), decltype(&HookDefaults::initialize)> &&
               std::is_same_v<decltype(&H::finalize), decltype(&HookDefaults::finalize)>;
}();

} // namespace odegpu

#endif
