"""Parity helpers shared by the GPU tests, smoke() and the parity report.

Runs a workload through the product (C ABI) and through a CPU checker on the
same inputs and compares with the rules of SURVEY.md §8(c):
* exact: accepted / rejected steps, event detections, stop reason, secant failures;
* <= rtol relative (absolute floor `atol`) on state, accessories, td, final_t;
* components pinned by a stop event (|F| <= event tol at the stop) compared
  with |d| <= 2 * event_tol instead;
* time-of-extremum accessories: within one local step (smallest_step) when
  the matching value accessory agrees.
"""
from __future__ import annotations

import numpy as np

import paper_1810_03931_b200 as pkg
from paper_1810_03931_b200 import abi

COUNT_FIELDS = ("accepted_steps", "rejected_steps", "event_detections", "reason", "secant_failures")


def run_gpu(wl, iterations: int, device: int = 0, trace: bool = False):
    td, y, p, acc = wl.arrays()
    pool = pkg.ProblemPool.from_arrays(td, y, p, acc)
    batch = pkg.SolverBatch(pkg.make_batch_dims(wl.n, wl.model.dims()), device=device)
    pkg.linear_set(batch, pool, pkg.LinearCopySpec(0, 0, wl.n))
    cfg = pkg.SolverConfig(wl.algorithm, wl.dt)
    tr = [] if trace else None

    def sink(it, b):
        tr.append(dict(td=b.time_domain(), y=b.state(), acc=b.accessories(), outcomes=b.outcomes()))

    pkg.solve_iteratively(batch, wl.model, cfg, iterations, sink if trace else None)
    out = dict(td=batch.time_domain(), y=batch.state(), acc=batch.accessories(), outcomes=batch.outcomes(),
               launches=batch.launch_count(), trace=tr)
    batch.close()
    return out


def rel_err(a, b, atol):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    both_nan = np.isnan(a) & np.isnan(b)
    same_inf = np.isinf(a) & np.isinf(b) & (np.sign(a) == np.sign(b))
    d = np.abs(a - b) / (np.abs(b) + atol)
    d[both_nan | same_inf] = 0.0
    d[np.isnan(d)] = np.inf
    return d


def compare(wl, gpu, ref, *, pinned_state=(), pinned_acc=(), time_acc=()) -> dict:
    """Per-field statistics; `pinned_*` are component indices compared with
    the event-tolerance rule, `time_acc` maps time-accessory -> value-accessory."""
    n = wl.n
    d = wl.model.dims()
    og, orf = gpu["outcomes"], ref["outcomes"]
    rep = {"n": n}
    for k in COUNT_FIELDS:
        rep[f"mismatch_{k}"] = int(np.count_nonzero(og[k] != orf[k]))
    atol = float(min(wl.model.ode_controls().abs_tol))
    ev_tol = max(wl.model.event_controls().tolerance or [0.0])
    stopped = orf["reason"] == abi.EVENT_STOP
    y_g = gpu["y"].reshape(d.system_dim, n)
    y_r = ref["y"].reshape(d.system_dim, n)
    worst = 0.0
    for c in range(d.system_dim):
        if c in pinned_state:
            e = np.abs(y_g[c] - y_r[c])
            rep[f"y{c}_pinned_abs"] = float(np.max(np.where(stopped, e, 0.0))) if n else 0.0
            free = ~stopped
            rep[f"y{c}_rel"] = float(np.max(rel_err(y_g[c][free], y_r[c][free], atol), initial=0.0))
        else:
            rep[f"y{c}_rel"] = float(np.max(rel_err(y_g[c], y_r[c], atol), initial=0.0))
        worst = max(worst, rep[f"y{c}_rel"])
    a_g = gpu["acc"].reshape(max(d.accessory_count, 1), n) if d.accessory_count else None
    a_r = ref["acc"].reshape(max(d.accessory_count, 1), n) if d.accessory_count else None
    for c in range(d.accessory_count):
        if c in time_acc:
            vc = time_acc[c]
            same_val = rel_err(a_g[vc], a_r[vc], atol) <= 1e-9
            step = np.where(np.isfinite(orf["smallest_step"]), orf["smallest_step"], 0.0)
            dt = np.abs(a_g[c] - a_r[c])
            rep[f"acc{c}_time_steps_off"] = int(np.count_nonzero(same_val & (dt > step * 1.000001 + 1e-15)))
            rep[f"acc{c}_time_rel_info"] = float(np.max(rel_err(a_g[c], a_r[c], atol), initial=0.0))
        elif c in pinned_acc:
            rep[f"acc{c}_pinned_abs"] = float(np.max(np.abs(a_g[c] - a_r[c]), initial=0.0))
        else:
            rep[f"acc{c}_rel"] = float(np.max(rel_err(a_g[c], a_r[c], atol), initial=0.0))
            worst = max(worst, rep[f"acc{c}_rel"])
    # Times located by the event machine (final_t of an EventStop, and t0
    # after BubbleCollapse's finalize) are pinned only by |F| <= tol: two
    # runs may stop anywhere inside the zone, |dt| <= 2 tol / |dF/dt|.
    ft_err = rel_err(og["final_t"], orf["final_t"], atol)
    td_err = rel_err(gpu["td"], ref["td"], atol).reshape(2, n)
    if ev_tol and stopped.any():
        slope = event_slope(wl, ref, np.nonzero(stopped)[0])
        allowed = 4.0 * ev_tol / np.maximum(slope, 1e-300)
        loc_ok = np.abs(og["final_t"][stopped] - orf["final_t"][stopped]) <= allowed
        rep["located_t_outside_zone_bound"] = int(np.count_nonzero(~loc_ok))
        ft_err[stopped] = 0.0
        td0_ok = np.abs(gpu["td"][:n][stopped] - ref["td"][:n][stopped]) <= allowed
        rep["located_t_outside_zone_bound"] += int(np.count_nonzero(~td0_ok))
        td_err[0, stopped] = 0.0
    rep["td_rel"] = float(np.max(td_err, initial=0.0))
    rep["final_t_rel"] = float(np.max(ft_err, initial=0.0))
    rep["event_tol"] = ev_tol
    rep["worst_rel"] = worst
    rep["steps"] = int(orf["accepted_steps"].sum() + orf["rejected_steps"].sum())
    return rep


def event_slope(wl, ref, idx):
    """|dF0/dt| at the reference's stop points; F0 = y2 for every stop event
    of the workloads (duffing.hpp:136, keller_miksis.hpp:324, valve.hpp:435),
    so dF0/dt = dy2/dt from the model RHS (evaluated by the C oracle, one
    batched call)."""
    import ctypes as C

    from oracle import pyoracle

    lib = pyoracle.load("port")
    d = wl.model.dims()
    n = wl.n
    k = idx.size
    y = np.ascontiguousarray(ref["y"].reshape(d.system_dim, n)[:, idx])
    p = (np.ascontiguousarray(wl.p.reshape(d.param_count, n)[:, idx]) if d.param_count else np.zeros(1))
    t = np.ascontiguousarray(ref["outcomes"]["final_t"][idx], dtype=np.float64)
    dy = np.zeros((d.system_dim, k))
    rc = lib.odo_rhs_batch(C.byref(wl.model.to_c()), k, abi.vptr(t), abi.vptr(y), abi.vptr(p), d.system_dim,
                           d.param_count, abi.vptr(dy))
    assert rc == 0
    return np.abs(dy[1])


# Per-config comparison rules: which components a stop event
# pins, which accessories are times of extrema.
RULES = {
    "cfg1_duffing_rk4": dict(time_acc={1: 0, 3: 2}),
    "cfg2_duffing_rkck45_event": dict(time_acc={1: 0}),
    "cfg3_keller_miksis": dict(pinned_state=(1,), time_acc={0: 1, 2: 3}),
    # y1_min sits on the seat (y1 = 0, impact zone |y1| <= tol) for impacting q
    "cfg4_valve": dict(pinned_state=(1,), pinned_acc=(1,), time_acc={}),
}
