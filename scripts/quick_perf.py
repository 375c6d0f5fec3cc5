"""Device time of one solve per config at full size (no torch): pristine batch
restored before each run, kernel time from CUDA events on the batch stream.
Usage: [ODEGPU_LIB=...] [FETCH=0|1|2] python scripts/quick_perf.py [cfg ...]"""
import json, os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1810_03931_b200 as pkg

peak, _ = pkg.dfma_peak()
lib = os.environ.get("ODEGPU_LIB", "default")
for name in sys.argv[1:] or ["cfg2", "cfg3", "cfg4", "cfg1"]:
    wl = pkg.workloads.CONFIGS[name]()
    td, y, p, acc = wl.arrays()
    pool = pkg.ProblemPool.from_arrays(td, y, p, acc)
    dims = pkg.make_batch_dims(wl.n, wl.model.dims())
    b, pristine = pkg.SolverBatch(dims), pkg.SolverBatch(dims)
    if "FETCH" in os.environ:  # abi.FETCH_* (default: the model's policy)
        b.set_fetch_order(int(os.environ["FETCH"]))
    pkg.linear_set(pristine, pool, pkg.LinearCopySpec(0, 0, wl.n))
    cfg = pkg.SolverConfig(wl.algorithm, wl.dt)
    runs = []
    for it in range(4):
        pkg.batch_copy(b, pristine)
        pkg.solve(b, wl.model, cfg)
        ms = b.last_kernel_ms()
        d = b.diagnostics()
        steps = d["accepted_steps"] + d["rejected_steps"]
        runs.append(dict(ms=round(ms, 3), steps=steps, frac=round(steps * wl.instr_per_step / (ms * 1e-3) / peak, 4)))
    best = min(runs[1:], key=lambda r: r["ms"])
    print(json.dumps(dict(lib=os.path.basename(lib), fetch=os.environ.get("FETCH", "auto"), name=name, n=wl.n, best_ms=best["ms"], steps=best["steps"],
                          steps_per_s=best["steps"] / best["ms"] * 1e3, frac=best["frac"], peak=peak)), flush=True)
    b.close(); pristine.close()
