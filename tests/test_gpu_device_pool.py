"""Device-resident pool (odegpu_device_pool_*): linear_set /
random_set from HBM equal the host-pool copies bit for bit, and the chunked,
cost-clustered pool solve (PAPER.md:833 re-batching) gives every system bit
for bit the result of one resident batch."""
import numpy as np
import pytest

import paper_1810_03931_b200 as pkg
from paper_1810_03931_b200 import abi, workloads

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a).view(np.uint64)


def test_random_set_from_device_pool_equals_host_pool():
    wl = workloads.CONFIGS["cfg4"]().strided(3000)
    td, y, p, acc = wl.arrays()
    pool = pkg.ProblemPool.from_arrays(td, y, p, acc)
    dpool = pkg.DevicePool.from_pool(pool)
    dims = pkg.make_batch_dims(1024, wl.model.dims())
    rng = np.random.default_rng(7)
    ib = rng.permutation(1024)[:700]
    ip = rng.choice(wl.n, 700, replace=False)
    for mode in (abi.COPY_ALL, abi.COPY_ACTUAL_STATE, abi.COPY_PARAMETER):
        a, b = pkg.SolverBatch(dims), pkg.SolverBatch(dims)
        pkg.random_set(a, pool, pkg.RandomCopySpec(ib, ip, mode))
        pkg.random_set_device(b, dpool, pkg.RandomCopySpec(ib, ip, mode))
        for get in ("time_domain", "state", "parameters", "accessories"):
            assert np.array_equal(bits(getattr(a, get)()), bits(getattr(b, get)())), (mode, get)
        assert a.outcomes().tobytes() == b.outcomes().tobytes()
        a.close(), b.close()
    # linear_set too, and the reference's validation
    a, b = pkg.SolverBatch(dims), pkg.SolverBatch(dims)
    pkg.linear_set(a, pool, pkg.LinearCopySpec(10, 500, 900))
    pkg.linear_set_device(b, dpool, pkg.LinearCopySpec(10, 500, 900))
    assert np.array_equal(bits(a.state()), bits(b.state()))
    with pytest.raises(pkg.OutOfRange, match="range exceeds batch capacity"):
        pkg.linear_set_device(b, dpool, pkg.LinearCopySpec(200, 0, 900))
    with pytest.raises(pkg.InvalidArgument, match="duplicate batch index 3"):
        pkg.random_set_device(b, dpool, pkg.RandomCopySpec([3, 3], [0, 1]))
    with pytest.raises(pkg.OutOfRange, match="pool index out of range"):
        pkg.random_set_device(b, dpool, pkg.RandomCopySpec([0], [wl.n]))
    a.close(), b.close()
    dpool.close()


def test_store_is_the_inverse_copy():
    wl = workloads.CONFIGS["cfg3"]().strided(2048)
    td, y, p, acc = wl.arrays()
    dpool = pkg.DevicePool.from_pool(pkg.ProblemPool.from_arrays(td, y, p, acc))
    b = pkg.SolverBatch(pkg.make_batch_dims(512, wl.model.dims()))
    rows = np.arange(100, 612)[::-1].copy()
    pkg.random_set_device(b, dpool, pkg.RandomCopySpec(np.arange(512), rows))
    pkg.solve(b, wl.model, pkg.SolverConfig(wl.algorithm, wl.dt))
    dpool.store(b, pkg.RandomCopySpec(np.arange(512), rows, abi.COPY_ACTUAL_STATE))
    y_pool = dpool.state().reshape(2, wl.n)
    y_b = b.state().reshape(2, 512)
    assert np.array_equal(bits(y_pool[:, rows]), bits(y_b))
    untouched = np.setdiff1d(np.arange(wl.n), rows)
    assert np.array_equal(bits(y_pool[:, untouched]), bits(y.reshape(2, wl.n)[:, untouched]))
    b.close(), dpool.close()


@pytest.mark.parametrize("cfg", ["cfg3", "cfg4"])
def test_clustered_pool_solve_equals_one_batch(cfg):
    wl = workloads.CONFIGS[cfg]().strided(12000)
    td, y, p, acc = wl.arrays()
    scfg = pkg.SolverConfig(wl.algorithm, wl.dt)
    ref = pkg.SolverBatch(pkg.make_batch_dims(wl.n, wl.model.dims()))
    pkg.linear_set(ref, pkg.ProblemPool.from_arrays(td, y, p, acc), pkg.LinearCopySpec(0, 0, wl.n))
    dpool = pkg.DevicePool.from_pool(pkg.ProblemPool.from_arrays(td, y, p, acc))
    # iteration 1 in pool order (no costs yet), 2-3 cost-clustered in chunks of 2500
    for it in range(3):
        pkg.solve(ref, wl.model, scfg)
        dpool.solve(wl.model, scfg, batch_capacity=2500, iterations=1, clustered=True)
        assert np.array_equal(bits(ref.time_domain()), bits(dpool.time_domain())), it
        assert np.array_equal(bits(ref.state()), bits(dpool.state())), it
        assert np.array_equal(bits(ref.accessories()), bits(dpool.accessories())), it
        assert ref.outcomes().tobytes() == dpool.outcomes().tobytes(), it
    # fused iterations inside the pool solve: the same as two more solves
    pkg.solve_iteratively(ref, wl.model, scfg, 2)
    dpool.solve(wl.model, scfg, batch_capacity=4096, iterations=2, clustered=True)
    assert np.array_equal(bits(ref.state()), bits(dpool.state()))
    assert ref.outcomes().tobytes() == dpool.outcomes().tobytes()
    ref.close(), dpool.close()


def test_pool_solve_rejects_t1_before_t0():
    wl = workloads.CONFIGS["cfg4"]().strided(1000)
    td, y, p, acc = wl.arrays()
    td = td.copy()
    td[1000 + 321] = -1.0  # t1 of system 321
    dpool = pkg.DevicePool.from_pool(pkg.ProblemPool.from_arrays(td, y, p, acc))
    with pytest.raises(pkg.InvalidArgument, match="system 321 has t1 < t0"):
        dpool.solve(wl.model, pkg.SolverConfig(wl.algorithm, wl.dt), batch_capacity=300)
    assert np.array_equal(bits(dpool.state()), bits(y))  # nothing integrated
    dpool.close()
