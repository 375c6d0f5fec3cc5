"""Fetch order (odegpu_batch_set_fetch_order): a scheduling hint only —
longest-first order must leave every value and count bitwise unchanged."""
import numpy as np
import pytest

import parity
import paper_1810_03931_b200 as pkg
from paper_1810_03931_b200 import abi, workloads

pytestmark = pytest.mark.gpu


def run(wl, mode, iterations):
    td, y, p, acc = wl.arrays()
    pool = pkg.ProblemPool.from_arrays(td, y, p, acc)
    b = pkg.SolverBatch(pkg.make_batch_dims(wl.n, wl.model.dims()))
    b.set_fetch_order(mode)
    pkg.linear_set(b, pool, pkg.LinearCopySpec(0, 0, wl.n))
    launches0 = b.launch_count()
    pkg.solve_iteratively(b, wl.model, pkg.SolverConfig(wl.algorithm, wl.dt), iterations)
    out = dict(td=b.time_domain(), y=b.state(), acc=b.accessories(), outcomes=b.outcomes(),
               launches=b.launch_count() - launches0)
    b.close()
    return out


@pytest.mark.parametrize("cfg", ["cfg2", "cfg3", "cfg4"])
def test_cost_order_changes_no_result(cfg):
    wl = workloads.CONFIGS[cfg]().strided(16384)
    nat, cost = run(wl, abi.FETCH_NATURAL, 3), run(wl, abi.FETCH_COST, 3)
    for k in ("td", "y", "acc"):
        assert np.array_equal(nat[k].view(np.uint64), cost[k].view(np.uint64)), k
    assert nat["outcomes"].tobytes() == cost["outcomes"].tobytes()
    # an order build (keys kernel) after each COST solve launch: one per
    # iteration, or a single one when the iterations run fused in one launch
    # (hooks.hpp kFusableIterations)
    assert nat["launches"] + 1 <= cost["launches"] <= nat["launches"] + 3


def test_auto_follows_the_model_policy():
    wl = workloads.CONFIGS["cfg1"]().strided(4096)  # RK4: natural under AUTO
    assert run(wl, abi.FETCH_AUTO, 2)["launches"] == run(wl, abi.FETCH_NATURAL, 2)["launches"]
    wl = workloads.CONFIGS["cfg4"]().strided(4096)  # adaptive valve: cost order
    assert run(wl, abi.FETCH_AUTO, 2)["launches"] == run(wl, abi.FETCH_COST, 2)["launches"]
    wl = workloads.CONFIGS["cfg3"]().strided(4096)  # Keller-Miksis: index order (models_keller_miksis.cu)
    assert run(wl, abi.FETCH_AUTO, 2)["launches"] == run(wl, abi.FETCH_NATURAL, 2)["launches"]


def test_rejects_unknown_mode():
    b = pkg.SolverBatch(pkg.BatchDims(8, 2, 4, 1, 2))
    with pytest.raises(pkg.InvalidArgument):
        b.set_fetch_order(7)
    b.close()


def test_scan_pipeline_rows_independent_of_fetch_order(monkeypatch):
    """Pipeline slots take their mode from ODEGPU_FETCH_ORDER at creation:
    a valve scan (iterations 2.. of every chunk longest-first under AUTO)
    gives bitwise the rows of the same scan in index order."""
    from paper_1810_03931_b200 import scan

    def run(mode):
        monkeypatch.setenv("ODEGPU_FETCH_ORDER", str(mode))
        spec = scan.ValveScanSpec(q=scan.ParamRange(0.2, 10.0, 6000), transient=24, saved=4,
                                  solver=scan.SolveOptions(rel_tol=1e-10, abs_tol=1e-10, batch_capacity=2048))
        return scan.run_valve_scan(spec)

    a, b = run(abi.FETCH_NATURAL), run(abi.FETCH_AUTO)
    assert a.rows.tobytes() == b.rows.tobytes()
    assert a.diagnostics == b.diagnostics
