"""Cost-clustered re-batching of a device-resident pool (odegpu_device_pool_solve):
the whole pool solved in chunks of `cap` systems, chunks in pool order vs cut
from the pool sorted longest first by the previous solve's cost.
Usage: python scripts/pool_cluster_perf.py [cfg3|cfg4|cfg5_22] [chunks]"""
import json, sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_1810_03931_b200 as pkg
from paper_1810_03931_b200 import workloads

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
chunks = int(sys.argv[2]) if len(sys.argv) > 2 else 8
wl = workloads.cfg5(int(name[5:])) if name.startswith("cfg5_") else workloads.CONFIGS[name]()
td, y, p, acc = wl.arrays()
pool = pkg.ProblemPool.from_arrays(td, y, p, acc)
cfg = pkg.SolverConfig(wl.algorithm, wl.dt)
cap = -(-wl.n // chunks)
peak, _ = pkg.dfma_peak()
for clustered in (False, True):
    dp = pkg.DevicePool.from_pool(pool)
    dp.solve(wl.model, cfg, cap, 1, clustered)  # iteration 0: gives the costs
    res = []
    for rep in range(3):  # iterations 1..3 in place, timed
        t0 = time.perf_counter()
        dp.solve(wl.model, cfg, cap, 1, clustered)
        dt = time.perf_counter() - t0
        o = dp.outcomes()
        steps = int(o["accepted_steps"].sum() + o["rejected_steps"].sum())
        res.append((dt, steps))
    dt = sum(r[0] for r in res); steps = sum(r[1] for r in res)
    print(json.dumps(dict(workload=wl.name, n=wl.n, chunks=chunks, clustered=clustered, ms_per_solve=dt / 3 * 1e3,
                          steps_per_s=steps / dt, frac=steps * wl.instr_per_step / dt / peak)), flush=True)
    dp.close()
# one resident batch, AUTO fetch order, same iterations, for scale
b = pkg.SolverBatch(pkg.make_batch_dims(wl.n, wl.model.dims()))
pkg.linear_set(b, pool, pkg.LinearCopySpec(0, 0, wl.n))
pkg.solve(b, wl.model, cfg)
t0 = time.perf_counter(); steps = 0
for rep in range(3):
    pkg.solve(b, wl.model, cfg)
    d = b.diagnostics(); steps += d["accepted_steps"] + d["rejected_steps"]
dt = time.perf_counter() - t0
print(json.dumps(dict(workload=wl.name, n=wl.n, chunks=1, resident_batch=True, ms_per_solve=dt / 3 * 1e3,
                      steps_per_s=steps / dt, frac=steps * wl.instr_per_step / dt / peak)), flush=True)
