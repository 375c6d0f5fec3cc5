"""Batch / pool / solve semantics through the CUDA path, mirroring the
reference's tests/test_pool.cpp and tests/test_batch.cpp."""
import math

import numpy as np
import pytest

import paper_1810_03931_b200 as pkg
from paper_1810_03931_b200 import abi, models
from paper_1810_03931_b200.api import InvalidArgument, OutOfRange

pytestmark = pytest.mark.gpu

TWO_PI = 2.0 * math.pi


def tagged_pool(n=16, dims=(2, 4, 3)):
    """test_pool.cpp:15-28: every slot holds a value encoding (array, system, component)."""
    s, p, a = dims
    pool = pkg.ProblemPool(pkg.PoolDims(n, s, p, a))
    for i in range(n):
        pool.set_time(i, 1000 + i, 2000 + i)
        for c in range(s):
            pool.set_state(i, c, 100 * c + i + 0.5)
        for c in range(p):
            pool.set_param(i, c, 10000 + 100 * c + i)
        for c in range(a):
            pool.set_accessory(i, c, -(100 * c + i) - 0.25)
    return pool


def duffing_pool(n, k_lo=0.2, k_hi=0.3):  # test_batch.cpp:18-33
    pool = pkg.ProblemPool(pkg.PoolDims(n, 2, 4, 0))
    for i in range(n):
        pool.set_time(i, 0.0, TWO_PI)
        k = k_lo if n == 1 else k_lo + (k_hi - k_lo) * i / (n - 1)
        for c, v in enumerate((k, 0.3, 1.0, 1.0)):
            pool.set_param(i, c, v)
    return pool


def new_batch(n, model):
    return pkg.SolverBatch(pkg.make_batch_dims(n, model.dims()))


def test_linear_set_all_and_round_trip():  # test_pool.cpp:69-107
    pool = tagged_pool(16)
    b = pkg.SolverBatch(pkg.BatchDims(16, 2, 4, 0, 3))
    pkg.linear_set(b, pool, pkg.LinearCopySpec(0, 0, 16))
    assert np.array_equal(b.time_domain(), pool.time_domain())
    assert np.array_equal(b.state(), pool.state())
    assert np.array_equal(b.parameters(), pool.parameters())
    assert np.array_equal(b.accessories(), pool.accessories())


def test_linear_set_single_property_touches_nothing_else():  # test_pool.cpp:78-98
    pool = tagged_pool(16)
    b = pkg.SolverBatch(pkg.BatchDims(8, 2, 4, 0, 3))
    pkg.linear_set(b, pool, pkg.LinearCopySpec(2, 5, 4, pkg.CopyMode.ActualState))
    st = b.state().reshape(2, 8)
    ps = pool.state().reshape(2, 16)
    assert np.array_equal(st[:, 2:6], ps[:, 5:9])
    assert np.all(st[:, :2] == 0) and np.all(st[:, 6:] == 0)
    assert np.all(b.time_domain() == 0) and np.all(b.parameters() == 0) and np.all(b.accessories() == 0)


def test_linear_set_rejects_bad_ranges():  # test_pool.cpp:109-120
    pool = tagged_pool(16)
    b = pkg.SolverBatch(pkg.BatchDims(8, 2, 4, 0, 3))
    with pytest.raises(OutOfRange):
        pkg.linear_set(b, pool, pkg.LinearCopySpec(4, 0, 5))
    with pytest.raises(OutOfRange):
        pkg.linear_set(b, pool, pkg.LinearCopySpec(0, 12, 5))
    with pytest.raises(OutOfRange):
        pkg.linear_set(b, pool, pkg.LinearCopySpec(-1, 0, 2))
    wrong = pkg.SolverBatch(pkg.BatchDims(8, 3, 4, 0, 3))
    with pytest.raises(InvalidArgument, match="disagree"):
        pkg.linear_set(wrong, pool, pkg.LinearCopySpec(0, 0, 2))


def test_random_set_places_and_rejects():  # test_pool.cpp:122-183
    pool = tagged_pool(16)
    b = pkg.SolverBatch(pkg.BatchDims(8, 2, 4, 0, 3))
    pkg.random_set(b, pool, pkg.RandomCopySpec([7, 0, 3], [2, 15, 2]))
    st = b.state().reshape(2, 8)
    ps = pool.state().reshape(2, 16)
    assert np.array_equal(st[:, 7], ps[:, 2]) and np.array_equal(st[:, 0], ps[:, 15])
    assert np.array_equal(st[:, 3], ps[:, 2])
    with pytest.raises(InvalidArgument, match="duplicate batch index 1"):
        pkg.random_set(b, pool, pkg.RandomCopySpec([1, 1], [0, 1]))
    with pytest.raises(OutOfRange):
        pkg.random_set(b, pool, pkg.RandomCopySpec([8], [0]))
    with pytest.raises(OutOfRange):
        pkg.random_set(b, pool, pkg.RandomCopySpec([0], [16]))
    with pytest.raises(InvalidArgument):
        pkg.random_set(b, pool, pkg.RandomCopySpec([0, 1], [0]))


def solved_state(pool, n):
    m = models.DuffingSystem()
    b = new_batch(n, m)
    pkg.linear_set(b, pool, pkg.LinearCopySpec(0, 0, n))
    pkg.solve(b, m, pkg.SolverConfig())
    return b


def test_solve_is_bitwise_deterministic_and_batch_independent():  # test_batch.cpp:85-112
    pool = duffing_pool(256)
    a = solved_state(pool, 256).state()
    assert np.array_equal(a, solved_state(pool, 256).state())
    # single-system batch equals the same system inside a full batch
    one = pkg.ProblemPool(pkg.PoolDims(1, 2, 4, 0))
    one.set_time(0, 0.0, TWO_PI)
    for c in range(4):
        one.set_param(0, c, pool.param_at(77, c))
    s = solved_state(one, 1).state()
    assert s[0] == a[77] and s[1] == a[77 + 256]


def test_permutation_identity():  # test_batch.cpp:114-139
    n = 64
    pool = duffing_pool(n)
    m = models.DuffingSystem()
    plain = solved_state(pool, n).state().reshape(2, n)
    perm = np.random.default_rng(42).permutation(n)
    b = new_batch(n, m)
    pkg.random_set(b, pool, pkg.RandomCopySpec(list(range(n)), perm.tolist()))
    pkg.solve(b, m, pkg.SolverConfig())
    st = b.state().reshape(2, n)
    assert np.array_equal(st, plain[:, perm])


def test_failure_isolation_and_sticky_abort():  # test_batch.cpp:139-167
    n = 32
    pool = duffing_pool(n)
    m = models.DuffingSystem()
    clean = solved_state(pool, n)
    poisoned = duffing_pool(n)
    poisoned.set_param(7, 1, float("nan"))
    dirty = new_batch(n, m)
    pkg.linear_set(dirty, poisoned, pkg.LinearCopySpec(0, 0, n))
    pkg.solve(dirty, m, pkg.SolverConfig())
    o = dirty.outcomes()
    assert o["reason"][7] == abi.NONFINITE_ABORT
    mask = np.arange(n) != 7
    assert np.array_equal(dirty.state().reshape(2, n)[:, mask], clean.state().reshape(2, n)[:, mask])
    assert np.all(o["reason"][mask] == abi.REACHED_END_TIME)
    before = dirty.state().copy()
    pkg.solve(dirty, m, pkg.SolverConfig())
    assert dirty.outcomes()["reason"][7] == abi.NONFINITE_ABORT
    st = dirty.state().reshape(2, n)
    assert st[0, 7] == before.reshape(2, n)[0, 7]  # skipped, untouched
    pkg.linear_set(dirty, pool, pkg.LinearCopySpec(7, 7, 1))
    assert dirty.outcomes()["reason"][7] == abi.REACHED_END_TIME


def test_empty_time_domain_in_a_batch():  # test_batch.cpp:171-182
    pool = duffing_pool(4)
    pool.set_time(0, 0.0, 0.0)
    pool.set_state(0, 0, 0.625)
    b = solved_state(pool, 4)
    o = b.outcomes()
    assert o["reason"][0] == abi.REACHED_END_TIME and o["accepted_steps"][0] == 0
    assert b.state_at(0, 0) == 0.625


def test_solve_rejects_inconsistent_setups():  # test_batch.cpp:184-204
    pool = duffing_pool(4)
    m = models.DuffingSystem()
    b = new_batch(4, m)
    pkg.linear_set(b, pool, pkg.LinearCopySpec(0, 0, 4))
    with pytest.raises(InvalidArgument, match="initial_time_step must be > 0"):
        pkg.solve(b, m, pkg.SolverConfig(initial_time_step=0.0))
    with pytest.raises(InvalidArgument, match="exceeds max_step"):
        pkg.solve(b, m, pkg.SolverConfig(initial_time_step=1e7))
    with pytest.raises(InvalidArgument, match="tile_size"):
        pkg.solve(b, m, pkg.SolverConfig(tile_size=0))
    wrong = pkg.SolverBatch(pkg.BatchDims(4, 3, 4, 0, 0))
    with pytest.raises(InvalidArgument, match="dimensions disagree"):
        pkg.solve(wrong, m, pkg.SolverConfig())
    backwards = duffing_pool(4)
    backwards.set_time(1, 0.0, -1.0)
    bb = new_batch(4, m)
    pkg.linear_set(bb, backwards, pkg.LinearCopySpec(0, 0, 4))
    before = bb.state().copy()
    with pytest.raises(InvalidArgument, match="system 1 has t1 < t0"):
        pkg.solve(bb, m, pkg.SolverConfig())
    assert np.array_equal(bb.state(), before)  # nothing was integrated
    with pytest.raises(InvalidArgument, match="iterations must be >= 1"):
        pkg.solve_iteratively(b, m, pkg.SolverConfig(), 0)


def test_solve_iteratively_sink_and_feed_forward():  # test_driver.cpp:183-234
    m = models.DuffingSystem()
    pool = duffing_pool(1, 0.215)
    b = new_batch(1, m)
    pkg.linear_set(b, pool, pkg.LinearCopySpec(0, 0, 1))
    points = []
    pkg.solve_iteratively(b, m, pkg.SolverConfig(), 1024 + 32,
                          lambda it, bb: points.append(bb.state_at(0, 0)) if it >= 1024 else None)
    assert len(points) == 32
    centers = []
    for v in points:
        if not any(abs(v - c) <= 1e-6 for c in centers):
            centers.append(v)
    assert len(centers) <= 4  # periodic window: a handful of section points


def test_hook_call_counts():  # test_driver.cpp:110-122
    m = models.CountingDef()
    pool = pkg.ProblemPool(pkg.PoolDims(1, 2, 4, 3))
    pool.set_time(0, 0.0, 5.0)
    pool.set_state(0, 0, 0.1)
    for c, v in enumerate((0.2, 0.3, 1.0, 1.0)):
        pool.set_param(0, c, v)
    b = new_batch(1, m)
    pkg.linear_set(b, pool, pkg.LinearCopySpec(0, 0, 1))
    pkg.solve(b, m, pkg.SolverConfig())
    acc = b.accessories()
    assert acc[0] == 1.0 and acc[1] == 1.0
    assert acc[2] == float(b.outcomes()["accepted_steps"][0])


def test_event_stop_on_local_maximum_and_equilibrium():  # test_events.cpp:184-277
    m = models.RampDef(1.0, 0.5, +1, 1)
    pool = pkg.ProblemPool(pkg.PoolDims(1, 1, 0, 0))
    pool.set_time(0, 0.0, 10.0)
    b = new_batch(1, m)
    pkg.linear_set(b, pool, pkg.LinearCopySpec(0, 0, 1))
    pkg.solve(b, m, pkg.SolverConfig())
    o = b.outcomes()
    assert o["reason"][0] == abi.EVENT_STOP and o["event_detections"][0] == 1
    assert o["final_t"][0] == pytest.approx(0.5, rel=1e-9) and abs(b.state_at(0, 0) - 0.5) <= 1e-6
    d = models.DecayDef()
    pool = pkg.ProblemPool(pkg.PoolDims(1, 1, 0, 0))
    pool.set_time(0, 0.0, 1e6)
    pool.set_state(0, 0, 1.0)
    b = new_batch(1, d)
    pkg.linear_set(b, pool, pkg.LinearCopySpec(0, 0, 1))
    pkg.solve(b, d, pkg.SolverConfig())
    o = b.outcomes()
    assert o["reason"][0] == abi.EQUILIBRIUM_STOP and o["event_detections"][0] == 1
    assert abs(b.state_at(0, 0)) <= 1e-6
