"""Warm-up solves and one profiled solve of a workload at full size (for ncu).

    python scripts/profile_one.py cfg2 [--n N] [--inplace K] [--log2n 24]

--inplace K: K in-place iterations (the bench's step, previous-iteration
fetch order) before the profiled one; ncu should then skip K+1 solve
launches (-s). Without it: one warm-up solve from the initial conditions and
one profiled solve from the initial conditions (cfg2's bench step)."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1810_03931_b200 as pkg  # noqa: E402
from paper_1810_03931_b200 import abi  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("name")
ap.add_argument("--n", type=int, default=0)
ap.add_argument("--inplace", type=int, default=-1)
ap.add_argument("--log2n", type=int, default=24)
args = ap.parse_args()
wl = pkg.workloads.cfg5(args.log2n) if args.name == "cfg5" else pkg.workloads.CONFIGS[args.name]()
if args.n:
    wl = wl.strided(args.n)
td, y, p, acc = wl.arrays()
pool = pkg.ProblemPool.from_arrays(td, y, p, acc)
b = pkg.SolverBatch(pkg.make_batch_dims(wl.n, wl.model.dims()))
pkg.linear_set(b, pool, pkg.LinearCopySpec(0, 0, wl.n))
cfg = pkg.SolverConfig(wl.algorithm, wl.dt)
if args.inplace >= 0:
    for _ in range(args.inplace + 1):
        pkg.solve(b, wl.model, cfg)
else:
    b.set_fetch_order(abi.FETCH_NATURAL)
    pristine = pkg.SolverBatch(pkg.make_batch_dims(wl.n, wl.model.dims()))
    pkg.batch_copy(pristine, b)
    pkg.solve(b, wl.model, cfg)
    pkg.batch_copy(b, pristine)
pkg.solve(b, wl.model, cfg)
d = b.diagnostics()
print(args.name, wl.n, d, "kernel ms", b.last_kernel_ms())
