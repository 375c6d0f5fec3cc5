"""Device detection log (odegpu_batch_set_detection_log) against the
reference's own on_detection observer (solve.hpp:46-50, driver.hpp:186-206)
run on the same inputs: the same detections, in the same per-system order,
with exact integer fields; times, values and states within the solver
parity tolerance."""
import numpy as np
import pytest

import paper_1810_03931_b200 as pkg
from oracle import pyoracle
from paper_1810_03931_b200 import abi, workloads

pytestmark = pytest.mark.gpu


def gpu_log(wl, capacity=None):
    td, y, p, acc = wl.arrays()
    pool = pkg.ProblemPool.from_arrays(td, y, p, acc)
    b = pkg.SolverBatch(pkg.make_batch_dims(wl.n, wl.model.dims()))
    b.set_detection_log(capacity if capacity is not None else 8 * wl.n)
    pkg.linear_set(b, pool, pkg.LinearCopySpec(0, 0, wl.n))
    pkg.solve(b, wl.model, pkg.SolverConfig(wl.algorithm, wl.dt))
    out = b.detection_log()
    oc = b.outcomes()
    b.close()
    return out, oc


@pytest.mark.parametrize("cfg,n", [("cfg2", 4096), ("cfg3", 2048), ("cfg4", 4096)])
def test_log_matches_reference_observer(cfg, n):
    wl = workloads.CONFIGS[cfg]().strided(n)
    (rec, pre, post, total), oc = gpu_log(wl)
    rrec, rpre, rpost, res = pyoracle.reference_detections(wl, 1)
    assert total == rec.size == rrec.size
    assert int(oc["event_detections"].sum()) == total
    for k in ("system", "event_index", "counter", "sequence", "kind", "in_zone"):
        assert np.array_equal(rec[k], rrec[k]), k
    # located points: the solver's parity tolerance: time and
    # state within 1e-9 relative; the event value within the zone's width
    scale = lambda a: np.abs(a) + 1e-9
    assert np.max(np.abs(rec["t"] - rrec["t"]) / scale(rrec["t"])) <= 1e-9
    tol = wl.model.event_controls().tolerance
    tol_of = np.asarray(tol)[rec["event_index"]]
    assert np.all(np.abs(rec["value"] - rrec["value"]) <= 2 * tol_of)
    # states at the located point: 1e-9 relative, with the absolute floor of
    # the components a stop event pins (|dy| <= 2 x event tolerance, the
    # parity rule of DESIGN.md §4)
    floor = 2 * float(np.max(tol))
    for a, b_ in ((pre, rpre), (post, rpost)):
        assert np.all(np.abs(a - b_) <= 1e-9 * np.abs(b_) + floor)


def test_log_overflow_counts_and_disables():
    wl = workloads.CONFIGS["cfg4"]().strided(1024)
    (rec, pre, post, total), oc = gpu_log(wl, capacity=100)
    assert rec.size == 100 and total == int(oc["event_detections"].sum()) > 100
    # disabling the log: plain solves again, and reading it is an error
    td, y, p, acc = wl.arrays()
    b = pkg.SolverBatch(pkg.make_batch_dims(wl.n, wl.model.dims()))
    b.set_detection_log(16)
    b.set_detection_log(0)
    pkg.linear_set(b, pkg.ProblemPool.from_arrays(td, y, p, acc), pkg.LinearCopySpec(0, 0, wl.n))
    pkg.solve(b, wl.model, pkg.SolverConfig(wl.algorithm, wl.dt))
    with pytest.raises(pkg.InvalidArgument):
        b.detection_log()
    b.close()


def test_log_leaves_results_unchanged():
    """The logging instantiation integrates bit for bit like the plain one."""
    wl = workloads.CONFIGS["cfg4"]().strided(2048)
    res = []
    for cap in (0, 1 << 16):
        td, y, p, acc = wl.arrays()
        b = pkg.SolverBatch(pkg.make_batch_dims(wl.n, wl.model.dims()))
        b.set_detection_log(cap)
        pkg.linear_set(b, pkg.ProblemPool.from_arrays(td, y, p, acc), pkg.LinearCopySpec(0, 0, wl.n))
        pkg.solve_iteratively(b, wl.model, pkg.SolverConfig(wl.algorithm, wl.dt), 3)
        res.append((b.state().copy(), b.accessories().copy(), b.outcomes().tobytes()))
        b.close()
    assert np.array_equal(res[0][0].view(np.uint64), res[1][0].view(np.uint64))
    assert np.array_equal(res[0][1].view(np.uint64), res[1][1].view(np.uint64))
    assert res[0][2] == res[1][2]
