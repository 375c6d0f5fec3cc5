"""One warm-up solve and one profiled solve of a workload at full size (for ncu).
Usage: python scripts/profile_one.py cfg2 [n]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1810_03931_b200 as pkg

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
wl = pkg.workloads.CONFIGS[name]()
if len(sys.argv) > 2:
    wl = wl.strided(int(sys.argv[2]))
td, y, p, acc = wl.arrays()
pool = pkg.ProblemPool.from_arrays(td, y, p, acc)
b = pkg.SolverBatch(pkg.make_batch_dims(wl.n, wl.model.dims()))
pkg.linear_set(b, pool, pkg.LinearCopySpec(0, 0, wl.n))
cfg = pkg.SolverConfig(wl.algorithm, wl.dt)
pkg.solve(b, wl.model, cfg)
pkg.solve(b, wl.model, cfg)
d = b.diagnostics()
print(name, wl.n, d, "kernel ms", b.last_kernel_ms())
