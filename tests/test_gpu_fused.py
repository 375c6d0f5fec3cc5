"""Fused iterations (solve_iteratively without a sink: each lane solves its
system `iterations` times in a row inside one kernel launch, for models whose
finalize keeps the time domain, include/odegpu/hooks.hpp kFusableIterations)
must equal `iterations` separate solve() calls bit for bit — time domains,
states, accessories, outcome records — and the batch's trial-step counter
must count every iteration."""
import numpy as np
import pytest

import paper_1810_03931_b200 as pkg
from paper_1810_03931_b200 import abi

pytestmark = pytest.mark.gpu


def load(wl, poison=None):
    td, y, p, acc = wl.arrays()
    if poison is not None:
        p = p.copy()
        p[poison] = np.nan  # parameter 0 of system `poison`: NonFiniteAbort, sticky
    pool = pkg.ProblemPool.from_arrays(td, y, p, acc)
    b = pkg.SolverBatch(pkg.make_batch_dims(wl.n, wl.model.dims()))
    pkg.linear_set(b, pool, pkg.LinearCopySpec(0, 0, wl.n))
    return b


def snapshot(b):
    o = b.outcomes()
    return [b.time_domain(), b.state(), b.accessories(), o.view(np.uint8)]


@pytest.mark.parametrize("name,n,its", [("cfg1", 1024, 5), ("cfg3", 2048, 4), ("cfg4", 2048, 6), ("cfg5", 0, 3)])
def test_fused_equals_separate_solves(name, n, its):
    wl = pkg.workloads.cfg5(14) if name == "cfg5" else pkg.workloads.CONFIGS[name]().strided(n)
    cfg = pkg.SolverConfig(wl.algorithm, wl.dt)
    fused = load(wl, poison=7)
    sep = load(wl, poison=7)
    fused.trial_steps(reset=True)
    launches0 = fused.launch_count()
    pkg.solve_iteratively(fused, wl.model, cfg, its)
    solve_launches = fused.launch_count() - launches0
    total = 0
    for _ in range(its):
        pkg.solve(sep, wl.model, cfg)
        o = sep.outcomes()
        live = o["reason"] != abi.NONFINITE_ABORT
        total += int(o["accepted_steps"][live].sum() + o["rejected_steps"][live].sum())
    for a, b in zip(snapshot(fused), snapshot(sep)):
        assert np.array_equal(a.view(np.uint8), b.view(np.uint8))
    assert fused.outcomes()["reason"][7] == abi.NONFINITE_ABORT
    # one solve kernel for all iterations (+ the t1 < t0 check, trig certificate, order build)
    assert solve_launches <= 4, solve_launches
    # every iteration's steps were counted (an aborted system's failed solve included)
    assert fused.trial_steps() >= total
