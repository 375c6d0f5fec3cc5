"""The reference's experiment protocols end to end (src/scan.cpp, the callers
of solve(): grid -> chunked pool -> transient + saved iterations -> rows),
odegpu's device pipeline vs the reference's own scan on all host threads,
same spec. Checks what tests/test_gpu_scan.py checks (parameter columns
bitwise, statuses and diagnostics counts exact) and reports wall times.
    python scripts/scan_bench.py > profiles/<tag>/scan_bench.jsonl"""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from oracle import pyoracle  # noqa: E402  (test infrastructure: the reference arm)
from paper_1810_03931_b200 import abi, scan  # noqa: E402

# (The Duffing maxima protocol iterated over many periods can meet the
# reference's own secant Zeno loop on some k — DESIGN.md §4 — so it is not
# benchmarked here.)
CASES = [
    ("bubble 512 PA1 x 512 f1, 8 transient + 4 saved collapses", abi.SCAN_BUBBLE,
     scan.BubbleScanSpec(pa1_bar=scan.ParamRange(0.5, 1.2, 512), pa2_bar=scan.ParamRange(0.0, 0.0, 1),
                         f1_khz=scan.ParamRange(20.0, 1000.0, 512, scan.LOG),
                         f2_khz=scan.ParamRange(20.0, 20.0, 1), transient=8, saved=4,
                         solver=scan.SolveOptions(rel_tol=1e-10, abs_tol=1e-10, batch_capacity=65536)),
     [0, 1, 2, 3]),
]

for name, protocol, spec, pcols in CASES:
    scan.run(protocol, spec)  # warm-up (module load, pinned staging)
    t0 = time.perf_counter()
    got = scan.run(protocol, spec)
    t_gpu = time.perf_counter() - t0
    t0 = time.perf_counter()
    rows, d = pyoracle.scan(protocol, spec)
    t_ref = time.perf_counter() - t0
    status = got.rows.shape[1] - 1
    g = got.diagnostics
    ok = (got.rows.shape == rows.shape and
          np.array_equal(got.rows[:, pcols].view(np.uint64), rows[:, pcols].view(np.uint64)) and
          np.array_equal(got.rows[:, status], rows[:, status]) and
          all(g[k] == d[k] for k in ("detections", "secant_failures", "nonfinite_systems", "reason_counts")))
    print(json.dumps(dict(scan=name, rows=int(rows.shape[0]), gpu_s=round(t_gpu, 4), reference_s=round(t_ref, 3),
                          reference_threads=pyoracle.host_cores(), speedup=round(t_ref / t_gpu, 1),
                          params_status_diagnostics_exact=bool(ok))), flush=True)
