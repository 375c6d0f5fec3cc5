"""Quick device timing of one solve per config at full size (CUDA events on the batch stream via torch)."""
import sys, time, json
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_1810_03931_b200 as pkg
peak, _ = pkg.dfma_peak()
for name in sys.argv[1:] or ["cfg2", "cfg3", "cfg4", "cfg1"]:
    wl = pkg.workloads.CONFIGS[name]()
    td, y, p, acc = wl.arrays()
    pool = pkg.ProblemPool.from_arrays(td, y, p, acc)
    b = pkg.SolverBatch(pkg.make_batch_dims(wl.n, wl.model.dims()))
    s = torch.cuda.Stream()
    b.set_stream(s.cuda_stream)
    pkg.linear_set(b, pool, pkg.LinearCopySpec(0, 0, wl.n))
    cfg = pkg.SolverConfig(wl.algorithm, wl.dt)
    pkg.solve(b, wl.model, cfg)  # warm-up
    res = []
    for it in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s); pkg.solve(b, wl.model, cfg); e1.record(s); e1.synchronize()
        ms = e0.elapsed_time(e1)
        o = b.outcomes()
        steps = int(o["accepted_steps"].sum() + o["rejected_steps"].sum())
        res.append(dict(ms=round(ms, 3), steps=steps, steps_per_s=steps / ms * 1e3,
                        frac=steps * wl.instr_per_step / (ms * 1e-3) / peak))
    print(json.dumps(dict(name=name, n=wl.n, runs=res, peak_lane_dfma=peak)), flush=True)
    b.close()
