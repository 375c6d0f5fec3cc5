// core.hpp — scalar types, enums and the host/device annotation shared by
// the device kernels and the C++ host API.
//
// Mirrors /root/reference/proj/include/odensemble/types.hpp:8-15 and
// driver.hpp:17-22; hooks are annotated ODEGPU_HD so one definition compiles
// for the host (g++) and into the sm_100a kernels (nvcc).
#ifndef ODEGPU_CORE_HPP
#define ODEGPU_CORE_HPP

#include <cstdint>

#if defined(__CUDACC__)
#define ODEGPU_HD __host__ __device__
#define ODEGPU_INLINE __forceinline__
#else
#define ODEGPU_HD
#define ODEGPU_INLINE inline
#endif

namespace odegpu {

using Real = double;        // types.hpp:8
using Index = std::int64_t; // types.hpp:10

enum class Algorithm { RK4 = 0, RKCK45 = 1 }; // types.hpp:12-15

enum class StopReason : std::uint8_t { // driver.hpp:17-22
    ReachedEndTime = 0,
    EventStop = 1,
    EquilibriumStop = 2,
    NonFiniteAbort = 3
};

} // namespace odegpu

#endif
