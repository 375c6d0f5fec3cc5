// odegpu.hpp — umbrella header of the C++ host API (the drop-in for
// #include "odensemble/solve.hpp" + models). Plain C++20; links against
// libodegpu.so (C ABI, include/odegpu.h). Namespace odegpu mirrors
// odensemble (types, pool, batch, solve, models).
#ifndef ODEGPU_ODEGPU_HPP
#define ODEGPU_ODEGPU_HPP

#include "odegpu/batch.hpp"
#include "odegpu/core.hpp"
#include "odegpu/models/duffing.hpp"
#include "odegpu/models/keller_miksis.hpp"
#include "odegpu/models/valve.hpp"
#include "odegpu/pool.hpp"
#include "odegpu/solve.hpp"
#include "odegpu/system.hpp"

#endif
