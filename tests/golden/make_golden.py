"""Generate the golden fixtures from the UNMODIFIED reference solver.

Runs oracle/_ref/libodref.so (the reference's own solve_iteratively compiled
from /root/reference/proj by oracle/Makefile) on small, evenly strided samples
of every SURVEY.md §8(d) workload and on the reference test-suite's fake
models, and stores inputs + outputs as compressed .npz files next to this
script. Only needed when /root/reference is present (this container); the
fixtures themselves are committed and travel to the GPU box.

    make ref && python tests/golden/make_golden.py
"""
from __future__ import annotations

import math
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))

from oracle import pyoracle  # noqa: E402
from paper_1810_03931_b200 import abi, models, workloads  # noqa: E402

TWO_PI = 2.0 * math.pi

# (fixture name, workload factory, sample size, iterations)
CONFIG_CASES = [
    ("cfg1", workloads.cfg1, 384, 3),
    ("cfg2", workloads.cfg2, 512, 2),
    ("cfg3", workloads.cfg3, 384, 3),
    ("cfg4", workloads.cfg4, 384, 4),
]


def save(name, model, algorithm, dt, iterations, td, y, p, acc, outcomes_in=None):
    inputs = dict(td=td.copy(), y=y.copy(), p=p.copy(), acc=acc.copy())
    oc, _, tr = pyoracle.solve("reference", model, td, y, p, acc, algorithm=algorithm, dt=dt,
                               iterations=iterations, outcomes=outcomes_in, trace=True)
    np.savez_compressed(
        HERE / f"{name}.npz",
        model_id=np.int32(model.model_id), consts=np.array(model.consts + [0.0] * (8 - len(model.consts))),
        algorithm=np.int32(algorithm), dt=np.float64(dt), iterations=np.int64(iterations),
        in_td=inputs["td"], in_y=inputs["y"], in_p=inputs["p"], in_acc=inputs["acc"],
        in_outcomes=outcomes_in if outcomes_in is not None else abi.empty_outcomes(td.size // 2),
        keep_outcomes=np.int8(outcomes_in is not None),
        td=td, y=y, acc=acc, outcomes=oc,
        trace_td=tr["td"], trace_y=tr["state"], trace_acc=tr["acc"], trace_outcomes=tr["outcomes"],
    )
    print(f"{name}: n={td.size // 2} iters={iterations} steps={int(oc['accepted_steps'].sum())} "
          f"reasons={np.bincount(oc['reason'], minlength=4).tolist()}")


def fakes():
    """Known-answer cases of the reference tests (tests/test_driver.cpp,
    tests/test_events.cpp, tests/test_batch.cpp), one system each."""
    one = lambda *v: np.array(v, dtype=np.float64)
    cases = [
        # test_driver.cpp:48-59 rk4 lands exactly on t1 with 4 steps
        ("fake_unit_slope_rk4", models.UnitSlopeDef(), abi.RK4, 0.25, one(0.0, 1.0), one(0.0), one(), one()),
        # test_driver.cpp:84-94 empty time domain
        ("fake_unit_slope_empty", models.UnitSlopeDef(), abi.RKCK45, 1e-3, one(2.5, 2.5), one(7.0), one(), one()),
        # test_events.cpp:184-197 stop at the first detection
        ("fake_ramp_stop", models.RampDef(1.0, 0.5, +1, 1), abi.RKCK45, 1e-3, one(0.0, 10.0), one(0.0), one(), one()),
        # test_events.cpp:199-210 equilibrium timeout
        ("fake_decay_equilibrium", models.DecayDef(), abi.RKCK45, 1e-3, one(0.0, 1e6), one(1.0), one(), one()),
        # test_events.cpp:212-225 start inside the zone
        ("fake_ramp_initial_in_zone", models.RampDef(1.0, 0.0, 0, 1), abi.RKCK45, 1e-3, one(0.0, 2.0), one(0.0),
         one(), one()),
        # test_events.cpp:227-238 single crossing counted once
        ("fake_ramp_single_crossing", models.RampDef(-1.0, 0.0, 0, 0), abi.RKCK45, 1e-3, one(0.0, 3.0), one(1.0),
         one(), one()),
        # test_events.cpp:240-251 wrong direction ignored
        ("fake_ramp_wrong_direction", models.RampDef(1.0, 0.5, -1, 1), abi.RKCK45, 1e-3, one(0.0, 2.0), one(0.0),
         one(), one()),
        # test_driver.cpp:110-122 hook call counts
        ("fake_counting", models.CountingDef(), abi.RKCK45, 1e-3, one(0.0, 5.0), one(0.1, 0.0),
         one(0.2, 0.3, 1.0, 1.0), one(0.0, 0.0, 0.0)),
        # test_driver.cpp:96-108 duffing event stop on a local maximum
        ("fake_duffing_event_stop", models.DuffingMaxEventSystem(1e-6, 1), abi.RKCK45, 1e-3, one(0.0, 1e6),
         one(0.3, 0.7), one(0.2, 0.3, 1.0, 1.0), one(0.0, 0.0)),
        # test_events.cpp:253-277 located point within tolerance
        ("fake_duffing_event_located", models.DuffingMaxEventSystem(1e-6, 1), abi.RKCK45, 1e-3, one(0.0, 100.0),
         one(0.1, 0.4), one(0.2, 0.3, 1.0, 1.0), one(0.0, 0.0)),
        # test_driver.cpp:61-82 adaptive run lands on t1
        ("fake_duffing_adaptive", models.DuffingSystem(), abi.RKCK45, 1e-3, one(0.0, TWO_PI), one(0.1, 0.0),
         one(0.2, 0.3, 1.0, 1.0), one()),
        # test_steppers.cpp:198-211 non-finite -> NonFiniteAbort at min step
        ("fake_blowup", models.BlowUpDef(), abi.RKCK45, 1e-3, one(0.0, 1.0), one(1.0), one(), one()),
        ("fake_blowup_rk4", models.BlowUpDef(), abi.RK4, 1e-3, one(0.0, 1.0), one(1.0), one(), one()),
        # valve seat contact (test_events.cpp:56-68 model) stopping at the seat
        ("fake_seat_contact", models.SeatContactDef(), abi.RKCK45, 1e-3, one(0.0, 10.0), one(0.5, -2.0, 10.0),
         one(1.25, 10.0, 20.0, 0.3, 0.8), one()),
        # RK4 + events: secant with RK4 re-steps
        ("fake_ramp_rk4_secant", models.RampDef(1.0, 0.35, 0, 1), abi.RK4, 0.1, one(0.0, 2.0), one(0.0), one(),
         one()),
    ]
    for name, model, alg, dt, td, y, p, acc in cases:
        save(name, model, alg, dt, 1, td, y, p, acc)


def batch_cases():
    """test_batch.cpp: a 32-system Duffing pool with one NaN parameter
    (failure isolation, :139-167) and a sticky-abort second solve."""
    n = 32
    k = np.array([0.2 + (0.3 - 0.2) * i / (n - 1) for i in range(n)])
    td = np.concatenate([np.zeros(n), np.full(n, TWO_PI)])
    y = np.zeros(2 * n)
    p = np.concatenate([k, np.full(n, 0.3), np.ones(n), np.ones(n)])
    p[7 + n] = np.nan  # forcing amplitude of system 7
    save("batch_nan_isolation", models.DuffingSystem(), abi.RKCK45, 1e-3, 2, td, y, p, np.zeros(0))
    # an empty time domain in a batch (test_batch.cpp:171-182)
    td2 = td.copy()
    td2[n] = td2[0]
    y2 = y.copy()
    y2[0] = 0.625
    p2 = np.concatenate([k, np.full(n, 0.3), np.ones(n), np.ones(n)])
    save("batch_empty_domain", models.DuffingSystem(), abi.RKCK45, 1e-3, 1, td2, y2, p2, np.zeros(0))
    # Lyapunov model (duffing.hpp:162-180): sample-and-reset finalize
    m = 64
    kk = np.array([0.2 + 0.1 * i / (m - 1) for i in range(m)])
    tdl = np.concatenate([np.zeros(m), np.full(m, TWO_PI)])
    yl = np.concatenate([np.zeros(m), np.zeros(m), np.ones(m), np.zeros(m)])
    pl = np.concatenate([kk, np.full(m, 0.3), np.ones(m), np.ones(m)])
    save("lyapunov", models.DuffingLyapunovSystem(), abi.RKCK45, 1e-3, 3, tdl, yl, pl, np.zeros(m))
    # RKCK45 Keller-Miksis without events, one forcing period
    wl = workloads.cfg3().strided(128)
    tdk, yk, pk, _ = wl.arrays()
    tdk[wl.n:] = 1.0
    save("keller_miksis_plain", models.KellerMiksisSystem(), abi.RKCK45, 1e-3, 1, tdk, yk, pk, np.zeros(0))


def main():
    if not pyoracle.available("reference"):
        sys.exit("oracle/_ref/libodref.so missing: run `make ref` (needs /root/reference)")
    for name, mk, count, its in CONFIG_CASES:
        wl = mk().strided(count)
        td, y, p, acc = wl.arrays()
        save(name, wl.model, wl.algorithm, wl.dt, its, td, y, p, acc)
    fakes()
    batch_cases()


if __name__ == "__main__":
    main()
