"""Exact-parity build vs the unmodified reference on seeded random off-grid
inputs (tests/test_gpu_random_parity.py's generator), many seeds: every array
of every system compared bit for bit after each of 3 iterations.
    ODEGPU_BUILD=parity python scripts/random_parity_sweep.py [seeds] [n]"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import numpy as np  # noqa: E402

from paper_1810_03931_b200 import abi  # noqa: E402
from oracle import pyoracle  # noqa: E402
import parity  # noqa: E402
from test_gpu_random_parity import make  # noqa: E402

assert abi.load().odegpu_build_flags() & abi.BUILD_PARITY, "run with ODEGPU_BUILD=parity"
seeds = int(sys.argv[1]) if len(sys.argv) > 1 else 10
n = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
total_sys = total_bad = 0
for case in ("duffing_event", "duffing_accessory", "duffing_rk4", "valve", "bubble"):
    for seed in range(seeds):
        wl = make(case, 90000 + 97 * seed + len(case)).strided(n)
        g = parity.run_gpu(wl, 3, trace=True)
        r = pyoracle.solve_workload("reference", wl, 3, trace=True)
        bad = np.zeros(wl.n, dtype=bool)
        for k in ("td", "y", "acc"):
            a, b = np.asarray(g[k]).reshape(-1, wl.n), np.asarray(r[k]).reshape(-1, wl.n)
            if a.size:
                bad |= np.any(a.view(np.uint64) != b.view(np.uint64), axis=0)
        for k in parity.COUNT_FIELDS + ("final_t", "smallest_step"):
            a, b = g["outcomes"][k], r["outcomes"][k]
            bad |= (a.view(np.uint64) != b.view(np.uint64)) if a.dtype.kind == "f" else (a != b)
        counts_per_it = [int(sum(np.count_nonzero(g["trace"][it]["outcomes"][k] !=
                                                  r["trace"]["outcomes"].reshape(3, wl.n)[it][k])
                                 for k in parity.COUNT_FIELDS)) for it in range(3)]
        total_sys += wl.n
        total_bad += int(bad.sum())
        print(json.dumps(dict(case=case, seed=seed, n=wl.n, iterations=3, bitwise_differing_systems=int(bad.sum()),
                              count_mismatches_per_iteration=counts_per_it)), flush=True)
print(json.dumps(dict(total_systems=total_sys, total_bitwise_differing=total_bad)), flush=True)
