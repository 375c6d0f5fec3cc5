// scan.cu — C ABI of the scan protocols (include/odegpu/scan.hpp, the
// reference's src/scan.cpp on the device pipeline): converts the C specs to
// the C++ ones and flattens ScanResult rows.
#include <cstring>

#include "internal.cuh"
#include "odegpu/scan.hpp"

using namespace odegpu;
using odegpu::detail::guarded;
using odegpu::detail::throw_invalid;
using odegpu::detail::throw_range;

namespace {

scan::ParamRange range_of(const odegpu_param_range& r) {
    return scan::ParamRange{r.min, r.max, r.res, r.log_scale ? scan::Scale::Log : scan::Scale::Linear};
}

scan::SolveOptions options_of(const odegpu_scan_options& o) {
    scan::SolveOptions s;
    if (o.algorithm != ODEGPU_RK4 && o.algorithm != ODEGPU_RKCK45) throw_invalid("scan: unknown algorithm");
    s.algorithm = o.algorithm == ODEGPU_RK4 ? Algorithm::RK4 : Algorithm::RKCK45;
    s.dt = o.dt;
    s.rel_tol = o.rel_tol;
    s.abs_tol = o.abs_tol;
    s.event_tol = o.event_tol;
    s.batch_capacity = o.batch_capacity;
    s.device = o.device;
    if (o.n_devices > 0 && !o.devices) throw_invalid("scan: n_devices > 0 without devices");
    for (int32_t d = 0; d < o.n_devices; ++d) s.devices.push_back(o.devices[d]);
    return s;
}

scan::DuffingScanSpec duffing_of(const odegpu_duffing_scan& d) {
    scan::DuffingScanSpec s;
    s.k = range_of(d.k);
    s.forcing_amplitude = d.forcing_amplitude;
    s.stiffness = d.stiffness;
    s.forcing_omega = d.forcing_omega;
    s.ic = {d.ic[0], d.ic[1]};
    s.transient = d.transient;
    s.saved = d.saved;
    s.solver = options_of(d.solver);
    return s;
}

scan::BubbleScanSpec bubble_of(const odegpu_bubble_scan& b) {
    scan::BubbleScanSpec s;
    s.pa1_bar = range_of(b.pa1_bar);
    s.pa2_bar = range_of(b.pa2_bar);
    s.f1_khz = range_of(b.f1_khz);
    s.f2_khz = range_of(b.f2_khz);
    s.material.R_E = b.R_E;
    s.material.c_L = b.c_L;
    s.material.rho_L = b.rho_L;
    s.material.P_inf = b.P_inf;
    s.material.p_V = b.p_V;
    s.material.sigma = b.sigma;
    s.material.mu_L = b.mu_L;
    s.material.gamma = b.gamma;
    s.material.theta = b.theta;
    s.ic = {b.ic[0], b.ic[1]};
    s.t_end = b.t_end;
    s.transient = b.transient;
    s.saved = b.saved;
    s.solver = options_of(b.solver);
    return s;
}

scan::ValveScanSpec valve_of(const odegpu_valve_scan& v) {
    scan::ValveScanSpec s;
    s.q = range_of(v.q);
    s.kappa = v.kappa;
    s.delta = v.delta;
    s.beta = v.beta;
    s.restitution = v.restitution;
    s.ic = {v.ic[0], v.ic[1], v.ic[2]};
    s.t_end = v.t_end;
    s.transient = v.transient;
    s.saved = v.saved;
    s.solver = options_of(v.solver);
    return s;
}

/// C++ exceptions of the host API (std::invalid_argument etc.) as ABI codes.
template <class F>
scan::ScanResult call(F&& f) {
    try {
        return f();
    } catch (const odegpu::detail::Error&) {
        throw;
    } catch (const std::out_of_range& e) {
        throw_range(e.what());
    } catch (const std::invalid_argument& e) {
        throw_invalid(e.what());
    }
}

} // namespace

extern "C" int odegpu_scan_run(int32_t protocol, const void* spec, double* rows, odegpu_index max_rows,
                               odegpu_index* n_rows, odegpu_index* n_columns, odegpu_scan_diagnostics* diag,
                               const char* output) {
    return guarded([&] {
        if (!spec || !n_rows || !n_columns) throw_invalid("scan: null argument");
        const std::string out = output ? output : "";
        scan::ScanResult r;
        switch (protocol) {
        case ODEGPU_SCAN_DUFFING_POINCARE:
        case ODEGPU_SCAN_DUFFING_MAXIMA_ACCESSORY:
        case ODEGPU_SCAN_DUFFING_MAXIMA_EVENT:
        case ODEGPU_SCAN_DUFFING_LYAPUNOV: {
            auto s = duffing_of(*static_cast<const odegpu_duffing_scan*>(spec));
            s.output = out;
            r = call([&] {
                if (protocol == ODEGPU_SCAN_DUFFING_POINCARE) return scan::run_duffing_poincare(s);
                if (protocol == ODEGPU_SCAN_DUFFING_LYAPUNOV) return scan::run_duffing_lyapunov(s);
                return scan::run_duffing_maxima(s, protocol == ODEGPU_SCAN_DUFFING_MAXIMA_EVENT
                                                       ? scan::MaximaMode::Event
                                                       : scan::MaximaMode::Accessory);
            });
            break;
        }
        case ODEGPU_SCAN_BUBBLE: {
            auto s = bubble_of(*static_cast<const odegpu_bubble_scan*>(spec));
            s.output = out;
            r = call([&] { return scan::run_bubble_scan(s); });
            break;
        }
        case ODEGPU_SCAN_VALVE: {
            auto s = valve_of(*static_cast<const odegpu_valve_scan*>(spec));
            s.output = out;
            r = call([&] { return scan::run_valve_scan(s); });
            break;
        }
        default:
            throw_invalid("scan: unknown protocol");
        }
        const Index nr = std::ssize(r.rows), nc = std::ssize(r.columns);
        *n_rows = nr;
        *n_columns = nc;
        if (rows) {
            if (max_rows < nr) throw_range("scan: rows buffer holds " + std::to_string(max_rows) + " rows, needs " +
                                           std::to_string(nr));
            for (Index i = 0; i < nr; ++i)
                std::memcpy(rows + i * nc, r.rows[static_cast<std::size_t>(i)].data(), size_t(nc) * 8);
        }
        if (diag) {
            const auto& d = r.diagnostics;
            *diag = odegpu_scan_diagnostics{};
            diag->detections = d.detections;
            diag->detections_outside_zone = d.detections_outside_zone;
            diag->max_residual_ratio = d.max_residual_ratio;
            diag->secant_failures = d.secant_failures;
            diag->nonfinite_systems = d.nonfinite_systems;
            for (int k = 0; k < 4; ++k) diag->reason_counts[k] = d.reason_counts[static_cast<std::size_t>(k)];
            diag->start_times_strictly_increase = d.start_times_strictly_increase ? 1 : 0;
        }
    });
}

extern "C" int odegpu_param_range_values(const odegpu_param_range* range, double* out) {
    return guarded([&] {
        if (!range || !out) throw_invalid("param_range_values: null argument");
        const auto v = call([&] {
            scan::ScanResult r;
            r.rows.push_back(range_of(*range).values());
            return r;
        });
        std::memcpy(out, v.rows[0].data(), v.rows[0].size() * 8);
    });
}
