"""e2e (host buffers through odegpu_pipeline_run) vs chunk count: python scripts/e2e_chunks.py [cfg] [chunks...]"""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_1810_03931_b200 as pkg
from paper_1810_03931_b200 import abi, workloads
cfg = sys.argv[1] if len(sys.argv) > 1 else 'cfg2'
wl = workloads.cfg5(int(cfg[5:].lstrip('_') or 24)) if cfg.startswith('cfg5') else workloads.CONFIGS[cfg]()
n = wl.n
td, y, p, acc = wl.arrays()
pin = lambda a: torch.from_numpy(a).pin_memory().numpy()
pool = pkg.ProblemPool.from_arrays(td, y, p, acc)
pool._td, pool._state, pool._params, pool._acc = pin(td), pin(y), pin(p), pin(acc)
outs = (pin(np.zeros(2 * n)), pin(np.zeros(y.size)), pin(np.zeros(acc.size)),
        torch.zeros(n * abi.OUTCOME_DTYPE.itemsize, dtype=torch.uint8, pin_memory=True).numpy().view(abi.OUTCOME_DTYPE))
cfg = pkg.SolverConfig(wl.algorithm, wl.dt)
for chunks in [int(a) for a in sys.argv[2:]] or (4, 8, 12, 16):
    pipe = pkg.api.Pipeline(wl.model, n // chunks, 0)
    pipe.run(pool, cfg, 1, out_arrays=outs)
    best = 1e9
    for _ in range(3):
        t0 = time.perf_counter(); pipe.run(pool, cfg, 1, out_arrays=outs); best = min(best, time.perf_counter() - t0)
    steps = int(outs[3]["accepted_steps"].sum() + outs[3]["rejected_steps"].sum())
    print(f"chunks {chunks:3d}: {best*1e3:7.3f} ms  e2e {steps/best:.4e} steps/s", flush=True)
    pipe.close()
