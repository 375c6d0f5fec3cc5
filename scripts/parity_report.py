"""GPU-vs-oracle parity report over the four configs at several horizons.
Usage (GPU box): python scripts/parity_report.py [--n 4096]"""
import argparse, json, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import numpy as np
import paper_1810_03931_b200 as pkg
from oracle import pyoracle
import parity

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=4096)
ap.add_argument("--iters", default="1,4")
args = ap.parse_args()
for name, mk in pkg.workloads.CONFIGS.items():
    wl = mk().strided(args.n)
    for its in [int(x) for x in args.iters.split(",")]:
        t0 = time.time(); g = parity.run_gpu(wl, its); tg = time.time() - t0
        r = pyoracle.solve_workload("port", wl, its)
        rep = parity.compare(wl, g, r, **parity.RULES[wl.name])
        rep.update(name=name, iterations=its, gpu_s=round(tg, 3), cpu_s=round(r["seconds"], 3))
        print(json.dumps(rep), flush=True)
        if any(rep[f"mismatch_{k}"] for k in parity.COUNT_FIELDS):
            og, orf = g["outcomes"], r["outcomes"]
            bad = np.nonzero((og["accepted_steps"] != orf["accepted_steps"]) | (og["event_detections"] != orf["event_detections"]) | (og["reason"] != orf["reason"]))[0][:5]
            for i in bad:
                print("  mismatch sys", int(i), {k: (int(og[k][i]), int(orf[k][i])) for k in parity.COUNT_FIELDS}, flush=True)
rate, secs = pkg.dfma_peak()
print(json.dumps({"dfma_lane_per_s": rate, "seconds": secs, "tflops": 2 * rate / 1e12}))
