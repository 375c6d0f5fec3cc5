"""Full-size parity gate: EVERY system of each BASELINE config, GPU build vs
the unmodified reference solver (oracle/_ref, all host threads).

    python scripts/parity_fullsize.py [--configs cfg1,cfg2,cfg3,cfg4,cfg5] [--out DIR]
    ODEGPU_BUILD=parity python scripts/parity_fullsize.py ...   # the -fmad=false build

Per config and iteration: exact accepted / rejected / detections / reason /
secant failures on every system (tests/parity.py COUNT_FIELDS), the value
rules of tests/parity.py, and the indices of every count mismatch (for
scripts/triage_count_mismatch.py). Reference results are cached under
/tmp/odegpu_parity_cache so the fast and parity builds (two processes) share
one reference run. Test infrastructure: runs the oracle, never shipped.
"""
import argparse
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import numpy as np  # noqa: E402

import paper_1810_03931_b200 as pkg  # noqa: E402
from paper_1810_03931_b200 import abi  # noqa: E402
from oracle import pyoracle  # noqa: E402
import parity  # noqa: E402

# config -> (workload factory, iterations compared): cfg1 over 16 forcing
# periods, cfg2 over 2 (its 3rd period holds the reference's own Zeno loop,
# DESIGN.md §4), cfg3/cfg4 two in-place iterations, cfg5 one.
PLAN = {
    "cfg1": (lambda: pkg.workloads.cfg1(), 16),
    "cfg2": (lambda: pkg.workloads.cfg2(), 2),
    "cfg3": (lambda: pkg.workloads.cfg3(), 2),
    "cfg4": (lambda: pkg.workloads.cfg4(), 2),
    "cfg5": (lambda: pkg.workloads.cfg5(24), 1),
}
CACHE = Path(os.environ.get("ODEGPU_PARITY_CACHE", "/tmp/odegpu_parity_cache"))


def reference(name, wl, its):
    f = CACHE / f"{name}_{wl.n}_{its}.npz"
    if f.exists():
        z = np.load(f)
        return dict(td=z["td"], y=z["y"], acc=z["acc"], outcomes=z["outcomes"], seconds=float(z["seconds"]),
                    trace=dict(outcomes=z["trace_outcomes"]) if "trace_outcomes" in z else None)
    workers = len(os.sched_getaffinity(0))
    r = pyoracle.solve_workload("reference", wl, its, trace=its > 1, workers=workers)
    CACHE.mkdir(parents=True, exist_ok=True)
    extra = {"trace_outcomes": r["trace"]["outcomes"]} if r["trace"] else {}
    np.savez(f, td=r["td"], y=r["y"], acc=r["acc"], outcomes=r["outcomes"], seconds=r["seconds"], **extra)
    return r


def gpu(wl, its):
    td, y, p, acc = wl.arrays()
    pool = pkg.ProblemPool.from_arrays(td, y, p, acc)
    batch = pkg.SolverBatch(pkg.make_batch_dims(wl.n, wl.model.dims()), device=0)
    pkg.linear_set(batch, pool, pkg.LinearCopySpec(0, 0, wl.n))
    cfg = pkg.SolverConfig(wl.algorithm, wl.dt)
    per_it = []
    t0 = time.time()
    pkg.solve_iteratively(batch, wl.model, cfg, its,
                          (lambda it, b: per_it.append(b.outcomes())) if its > 1 else None)
    secs = time.time() - t0
    out = dict(td=batch.time_domain(), y=batch.state(), acc=batch.accessories(), outcomes=batch.outcomes(),
               per_iteration=per_it, seconds=secs)
    batch.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="cfg1,cfg2,cfg3,cfg4,cfg5")
    ap.add_argument("--out", default=str(ROOT / "gpurun_out" / "parity_r02"))
    args = ap.parse_args()
    build = "parity" if abi.load().odegpu_build_flags() & abi.BUILD_PARITY else "fast"
    out_dir = Path(args.out)
    out_dir.mkdir(parents=True, exist_ok=True)
    log = open(out_dir / f"{build}.jsonl", "a")
    for name in args.configs.split(","):
        mk, its = PLAN[name]
        wl = mk()
        t0 = time.time()
        ref = reference(name, wl, its)
        t_ref = time.time() - t0
        g = gpu(wl, its)
        rep = parity.compare(wl, g, ref, **parity.RULES[wl.name])
        # bitwise: systems whose end state differs in any bit (any array)
        d = wl.model.dims()
        n = wl.n

        def differs(a, b, comps):
            a = np.asarray(a).reshape(comps, n).view(np.uint64)
            b = np.asarray(b).reshape(comps, n).view(np.uint64)
            return np.any(a != b, axis=0)

        bit = differs(g["td"], ref["td"], 2) | differs(g["y"], ref["y"], d.system_dim)
        if d.accessory_count:
            bit |= differs(g["acc"], ref["acc"], d.accessory_count)
        og, orf = g["outcomes"], ref["outcomes"]
        for k in ("final_t", "smallest_step"):
            bit |= og[k].view(np.uint64) != orf[k].view(np.uint64)
        rep["bitwise_differing_systems"] = int(bit.sum())
        rep.update(config=name, build=build, n=wl.n, iterations=its, ref_wall_s=round(t_ref, 2),
                   ref_solver_s=round(float(ref["seconds"]), 2), gpu_wall_s=round(g["seconds"], 3))
        # every iteration's integer counts (the end-of-run compare above covers the last)
        if its > 1 and ref.get("trace") is not None:
            tr = ref["trace"]["outcomes"].reshape(its, wl.n)
            per = []
            for it in range(its):
                og = g["per_iteration"][it]
                bad = np.zeros(wl.n, dtype=bool)
                for k in parity.COUNT_FIELDS:
                    bad |= og[k] != tr[it][k]
                per.append(int(bad.sum()))
                if bad.any():
                    rep.setdefault("mismatch_systems", {})[str(it)] = [
                        {"sys": int(i), **{k: [int(og[k][i]), int(tr[it][k][i])] for k in parity.COUNT_FIELDS}}
                        for i in np.nonzero(bad)[0][:50]]
            rep["count_mismatch_systems_per_iteration"] = per
        else:
            og, orf = g["outcomes"], ref["outcomes"]
            bad = np.zeros(wl.n, dtype=bool)
            for k in parity.COUNT_FIELDS:
                bad |= og[k] != orf[k]
            rep["count_mismatch_systems_per_iteration"] = [int(bad.sum())]
            if bad.any():
                rep["mismatch_systems"] = {"0": [
                    {"sys": int(i), **{k: [int(og[k][i]), int(orf[k][i])] for k in parity.COUNT_FIELDS}}
                    for i in np.nonzero(bad)[0][:50]]}
        line = json.dumps(rep)
        print(line, flush=True)
        log.write(line + "\n")
        log.flush()


if __name__ == "__main__":
    main()
