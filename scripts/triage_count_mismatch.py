"""Triage of integer mismatches GPU vs oracle on a strided BASELINE sample:
finds the systems whose counts differ, then re-runs each alone with the
tolerances scaled by (1 + eps) for small eps on BOTH sides — a count that
flips under a relative tolerance change far below the step-error noise marks an accept/reject or
zone decision sitting on a rounding tie (the 1-ulp libm / FMA-contraction
differences between the two builds decide it), not an algorithmic
difference; the FMA-contracted port (oracle/_build/libodeoracle_fma.so:
gcc -ffp-contract=fast -mfma) shows whether contraction alone moves it.
Usage (GPU box): python scripts/triage_count_mismatch.py cfg3 262144"""
import json, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import numpy as np
import parity
from oracle import pyoracle
from paper_1810_03931_b200 import workloads
from paper_1810_03931_b200.models import OdeControls

name, count = sys.argv[1], int(sys.argv[2])
wl = workloads.CONFIGS[name]().strided(count)
g = parity.run_gpu(wl, 1)
r = pyoracle.solve_workload("port", wl, 1)
og, orf = g["outcomes"], r["outcomes"]
bad = np.nonzero(np.logical_or.reduce([og[k] != orf[k] for k in parity.COUNT_FIELDS]))[0]
print(json.dumps(dict(config=name, systems=wl.n, mismatched=bad.tolist()[:20])), flush=True)


for i in bad[:5]:
    one = wl.subset(np.array([i]))
    row = dict(index=int(i), gpu={k: int(og[k][i]) for k in parity.COUNT_FIELDS},
               oracle={k: int(orf[k][i]) for k in parity.COUNT_FIELDS}, perturbed=[])
    base = one.model
    for eps in (-1e-7, -1e-8, -1e-9, -1e-10, -1e-12, 1e-12, 1e-10, 1e-9, 1e-8, 1e-7):
        tol = 1e-10 * (1 + eps)
        one.model = type(base)(1e-6, OdeControls.uniform(2, tol, tol)) if name == "cfg3" else base
        gg = parity.run_gpu(one, 1)["outcomes"]
        rr = pyoracle.solve_workload("port", one, 1)["outcomes"]
        row["perturbed"].append(dict(eps=eps, gpu_rejected=int(gg["rejected_steps"][0]),
                                     oracle_rejected=int(rr["rejected_steps"][0]),
                                     gpu_accepted=int(gg["accepted_steps"][0]),
                                     oracle_accepted=int(rr["accepted_steps"][0])))
    one.model = base
    # the port with FMA contraction (gcc -ffp-contract=fast -mfma, as nvcc
    # contracts the kernels), if built: oracle/_build/libodeoracle_fma.so
    fma = Path(pyoracle.PORT_LIB).with_name("libodeoracle_fma.so")
    if fma.exists():
        saved, pyoracle.PORT_LIB = pyoracle.PORT_LIB, fma
        pyoracle._libs.pop("port", None)
        rr = pyoracle.solve_workload("port", one, 1)["outcomes"]
        row["oracle_fma"] = {k: int(rr[k][0]) for k in parity.COUNT_FIELDS}
        pyoracle.PORT_LIB = saved
        pyoracle._libs.pop("port", None)
    print(json.dumps(row), flush=True)
