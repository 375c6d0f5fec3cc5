// pool.hpp — host problem pool and the shapes/copy specs of the C++ host
// API. Same names, layout and errors as the reference's
// /root/reference/proj/include/odensemble/pool.hpp:16-158: structure of
// arrays, component c of system i at [i + c * count].
#ifndef ODEGPU_POOL_HPP
#define ODEGPU_POOL_HPP

#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "odegpu.h"
#include "odegpu/core.hpp"
#include "odegpu/system.hpp"

namespace odegpu {

/// pool.hpp:16-23
inline Index flat_index(Index idx, Index component, Index count) {
    if (idx < 0 || idx >= count)
        throw std::out_of_range("flat_index: system index " + std::to_string(idx) + " outside [0, " +
                                std::to_string(count) + ")");
    if (component < 0) throw std::out_of_range("flat_index: negative component index");
    return component * count + idx;
}

/// pool.hpp:26-38
struct PoolDims {
    Index problem_size = 0, system_dim = 0, param_count = 0, accessory_count = 0;
    void validate() const {
        const char* what = problem_size < 1       ? "PoolDims: problem_size must be >= 1"
                           : system_dim < 1        ? "PoolDims: system_dim must be >= 1"
                           : param_count < 0       ? "PoolDims: param_count must be >= 0"
                           : accessory_count < 0   ? "PoolDims: accessory_count must be >= 0"
                                                   : nullptr;
        if (what) throw std::invalid_argument(what);
    }
};

/// pool.hpp:41-55
struct BatchDims {
    Index batch_capacity = 0, system_dim = 0, param_count = 0, event_count = 0, accessory_count = 0;
    void validate() const {
        const char* what = batch_capacity < 1     ? "BatchDims: batch_capacity must be >= 1"
                           : system_dim < 1        ? "BatchDims: system_dim must be >= 1"
                           : param_count < 0       ? "BatchDims: param_count must be >= 0"
                           : event_count < 0       ? "BatchDims: event_count must be >= 0"
                           : accessory_count < 0   ? "BatchDims: accessory_count must be >= 0"
                                                   : nullptr;
        if (what) throw std::invalid_argument(what);
    }
};

/// pool.hpp:65-69
inline BatchDims make_batch_dims(Index capacity, const SystemDims& sys) {
    BatchDims d{capacity, sys.system_dim, sys.param_count, sys.event_count, sys.accessory_count};
    d.validate();
    return d;
}

/// pool.hpp:142 (values equal the C-ABI odegpu_copy_mode)
enum class CopyMode { TimeDomain = 0, ActualState = 1, Parameter = 2, Accessories = 3, All = 4 };

/// pool.hpp:145-150
struct LinearCopySpec {
    Index start_in_batch = 0;
    Index start_in_pool = 0;
    Index element_count = 0;
    CopyMode copy_mode = CopyMode::All;
};

/// pool.hpp:154-158 (pool indices may repeat; batch indices must not)
struct RandomCopySpec {
    std::vector<Index> indices_in_batch;
    std::vector<Index> indices_in_pool;
    CopyMode copy_mode = CopyMode::All;
};

/// Host pool of all initial value problems (pool.hpp:74-139).
class ProblemPool {
public:
    explicit ProblemPool(const PoolDims& dims) : dims_(dims) {
        dims.validate();
        const auto n = static_cast<std::size_t>(dims.problem_size);
        arrays_[0].assign(2 * n, Real{0});
        arrays_[1].assign(static_cast<std::size_t>(dims.system_dim) * n, Real{0});
        arrays_[2].assign(static_cast<std::size_t>(dims.param_count) * n, Real{0});
        arrays_[3].assign(static_cast<std::size_t>(dims.accessory_count) * n, Real{0});
    }

    const PoolDims& dims() const { return dims_; }
    Index size() const { return dims_.problem_size; }

    std::span<Real> time_domain() { return arrays_[0]; }
    std::span<Real> state() { return arrays_[1]; }
    std::span<Real> parameters() { return arrays_[2]; }
    std::span<Real> accessories() { return arrays_[3]; }
    std::span<const Real> time_domain() const { return arrays_[0]; }
    std::span<const Real> state() const { return arrays_[1]; }
    std::span<const Real> parameters() const { return arrays_[2]; }
    std::span<const Real> accessories() const { return arrays_[3]; }

    Real& time_start(Index i) { return at(0, i, 0, 2, "time"); }
    Real& time_end(Index i) { return at(0, i, 1, 2, "time"); }
    Real time_start(Index i) const { return cat(0, i, 0, 2, "time"); }
    Real time_end(Index i) const { return cat(0, i, 1, 2, "time"); }
    Real& state_at(Index i, Index c) { return at(1, i, c, dims_.system_dim, "state"); }
    Real state_at(Index i, Index c) const { return cat(1, i, c, dims_.system_dim, "state"); }
    Real& param_at(Index i, Index c) { return at(2, i, c, dims_.param_count, "parameter"); }
    Real param_at(Index i, Index c) const { return cat(2, i, c, dims_.param_count, "parameter"); }
    Real& accessory_at(Index i, Index c) { return at(3, i, c, dims_.accessory_count, "accessory"); }
    Real accessory_at(Index i, Index c) const { return cat(3, i, c, dims_.accessory_count, "accessory"); }

    /// C-ABI view of the four arrays (odegpu_pool_view).
    odegpu_pool_view view() const {
        odegpu_pool_view v{};
        v.dims = {dims_.problem_size, dims_.system_dim, dims_.param_count, dims_.accessory_count};
        v.time_domain = arrays_[0].data();
        v.state = arrays_[1].data();
        v.parameters = arrays_[2].data();
        v.accessories = arrays_[3].data();
        return v;
    }

private:
    Real& at(int a, Index i, Index c, Index width, const char* what) {
        check(c, width, what);
        return arrays_[a][static_cast<std::size_t>(flat_index(i, c, size()))];
    }
    Real cat(int a, Index i, Index c, Index width, const char* what) const {
        check(c, width, what);
        return arrays_[a][static_cast<std::size_t>(flat_index(i, c, size()))];
    }
    static void check(Index c, Index width, const char* what) {
        if (c < 0 || c >= width) throw std::out_of_range(std::string("ProblemPool: ") + what + " component out of range");
    }

    PoolDims dims_;
    std::vector<Real> arrays_[4]; // time domain, state, parameters, accessories
};

} // namespace odegpu

#endif
