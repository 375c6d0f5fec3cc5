"""e2e through the pipeline in both modes with the per-chunk trace:
ODEGPU_PIPELINE_TRACE=1 python scripts/stream_trace.py cfg2 [cfg5_22 ...]"""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_1810_03931_b200 as pkg
from paper_1810_03931_b200 import abi, workloads
from paper_1810_03931_b200.api import PIPELINE_CHUNKED, PIPELINE_STREAMING, Pipeline, pinned

import os
no_oc = os.environ.get("NO_OUTCOMES") == "1"
modes = [int(m) for m in os.environ.get("MODES", "2,1").split(",")]
for name in sys.argv[1:] or ["cfg2"]:
    wl = workloads.cfg5(int(name[5:].lstrip('_') or 24)) if name.startswith('cfg5') else workloads.CONFIGS[name]()
    n = wl.n
    pool = pkg.ProblemPool.from_arrays(*wl.arrays()).pin()
    d = wl.model.dims()
    outs = (pinned(np.zeros(2 * n)), pinned(np.zeros(d.system_dim * n)), pinned(np.zeros(max(d.accessory_count, 1) * n)),
            None if no_oc else pinned(np.zeros(n, dtype=abi.OUTCOME_DTYPE)))
    cfg = pkg.SolverConfig(wl.algorithm, wl.dt)
    for mode in modes:
        # bench.py's chunking
        chunks = int(os.environ.get("CHUNKS", 0)) or int(min(max(round(n / 65536), 2), 16 if wl.instr_per_step > 500 else 8))
        pipe = Pipeline(wl.model, -(-n // chunks), 0, mode=mode)
        pipe.run(pool, cfg, 1, out_arrays=outs)
        best = 1e9
        for _ in range(3):
            print(f"--- {name} mode {mode}", file=sys.stderr, flush=True)
            t0 = time.perf_counter(); pipe.run(pool, cfg, 1, out_arrays=outs); best = min(best, time.perf_counter() - t0)
        if outs[3] is not None:
            steps = int(outs[3]["accepted_steps"].sum() + outs[3]["rejected_steps"].sum())
        print(f"{name} mode {mode}: {best*1e3:8.3f} ms  e2e {steps/best:.4e} steps/s", flush=True)
        pipe.close()
