"""Fetch-order effect in the scan-realistic setting: iteration 2 of an
in-place iterative solve (ordered by iteration 1's trial steps under
FETCH_COST) against the same iteration in natural order, plus the
same-solve-repeated setting bench.py uses. Kernel times (CUDA events).
Usage: python scripts/fetch_order_experiment.py [cfg ...]"""
import json, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1810_03931_b200 as pkg
from paper_1810_03931_b200 import abi

for name in sys.argv[1:] or ["cfg2", "cfg3", "cfg4"]:
    wl = pkg.workloads.CONFIGS[name]()
    td, y, p, acc = wl.arrays()
    pool = pkg.ProblemPool.from_arrays(td, y, p, acc)
    dims = pkg.make_batch_dims(wl.n, wl.model.dims())
    pristine = pkg.SolverBatch(dims)
    pkg.linear_set(pristine, pool, pkg.LinearCopySpec(0, 0, wl.n))
    cfg = pkg.SolverConfig(wl.algorithm, wl.dt)
    res = dict(name=name, n=wl.n)
    for mode, label in ((abi.FETCH_NATURAL, "natural"), (abi.FETCH_COST, "cost")):
        it2, rep = [], []
        for _ in range(3):
            b = pkg.SolverBatch(dims)
            b.set_fetch_order(mode)
            pkg.batch_copy(b, pristine)
            pkg.solve(b, wl.model, cfg)  # iteration 1 (natural: no costs yet)
            pkg.solve(b, wl.model, cfg)  # iteration 2, ordered by iteration 1
            it2.append(b.last_kernel_ms())
            pkg.batch_copy(b, pristine)  # the bench's setting: the same solve again
            pkg.solve(b, wl.model, cfg)
            rep.append(b.last_kernel_ms())
            b.close()
        res[f"iter2_{label}_ms"] = round(min(it2), 3)
        res[f"repeat_{label}_ms"] = round(min(rep), 3)
    print(json.dumps(res), flush=True)
