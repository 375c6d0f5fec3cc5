"""Bitwise comparison of two builds of libodegpu on the BASELINE workloads
(full size, a few iterations): proves that a kernel change that should not
alter any value (e.g. the time-term cache) does not.
Usage: [FETCH=0|1|2] python scripts/compare_libs.py run LIB OUT.npz [cfg ...]
       python scripts/compare_libs.py diff A.npz B.npz"""
import os, sys
from pathlib import Path
import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

if sys.argv[1] == "run":
    os.environ["ODEGPU_LIB"] = sys.argv[2]
    import parity
    import paper_1810_03931_b200 as pkg
    from paper_1810_03931_b200 import workloads
    if "FETCH" in os.environ:  # force a fetch order on every batch (abi.FETCH_*)
        init = pkg.SolverBatch.__init__

        def init_with_order(self, *a, **k):
            init(self, *a, **k)
            self.set_fetch_order(int(os.environ["FETCH"]))
        pkg.SolverBatch.__init__ = init_with_order
    out = {}
    for name in sys.argv[4:] or ["cfg1", "cfg2", "cfg3", "cfg4"]:
        import time
        t0 = time.time()
        wl = workloads.CONFIGS[name]().strided(int(os.environ.get("COMPARE_N", "65536")))
        r = parity.run_gpu(wl, 3)
        print(name, wl.n, f"{time.time() - t0:.1f}s", flush=True)
        for k in ("td", "y", "acc"):
            out[f"{name}_{k}"] = r[k]
        o = r["outcomes"]
        for k in o.dtype.names:
            out[f"{name}_out_{k}"] = np.ascontiguousarray(o[k])
    np.savez(sys.argv[3], **out)
else:
    a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
    bad = 0
    for k in sorted(a.files):
        x, y = a[k], b[k]
        same = np.array_equal(x.view(np.uint8), y.view(np.uint8)) if x.dtype.kind == "f" else np.array_equal(x, y)
        if not same:
            bad += 1
            n = int(np.sum(x != y)) if x.shape == y.shape else -1
            print(f"DIFF {k}: {n} elements differ")
    print(f"{len(a.files) - bad}/{len(a.files)} arrays bitwise identical")
