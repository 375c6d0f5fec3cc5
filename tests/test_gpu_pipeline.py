"""Chunked pool pipeline (odegpu_solve_pool / _multi): double-buffered chunks
must give bitwise the same results as one resident batch, because every
system's arithmetic depends only on its own data (solve.hpp:57-59)."""
import numpy as np
import pytest

import paper_1810_03931_b200 as pkg
from paper_1810_03931_b200 import abi, workloads

pytestmark = pytest.mark.gpu


def plain_run(wl, iterations, record_from):
    td, y, p, acc = wl.arrays()
    pool = pkg.ProblemPool.from_arrays(td, y, p, acc)
    b = pkg.SolverBatch(pkg.make_batch_dims(wl.n, wl.model.dims()))
    pkg.linear_set(b, pool, pkg.LinearCopySpec(0, 0, wl.n))
    snaps = []
    pkg.solve_iteratively(b, wl.model, pkg.SolverConfig(wl.algorithm, wl.dt), iterations,
                          lambda it, bb: snaps.append((bb.state(), bb.accessories(), bb.outcomes()))
                          if it >= record_from else None)
    return pool, dict(td=b.time_domain(), y=b.state(), acc=b.accessories(), outcomes=b.outcomes()), snaps


def outcome_bytes(o):
    raw = np.ascontiguousarray(o).view(np.uint8).reshape(-1, 56)
    return raw[:, [i for i in range(56) if not 9 <= i < 16]]


@pytest.mark.parametrize("cfg,count,cap,its,devices", [
    ("cfg4", 3000, 1024, 4, (0,)),
    ("cfg3", 2500, 1000, 3, (0,)),
    ("cfg2", 4097, 2048, 2, (0,)),
    ("cfg4", 3001, 700, 3, (0, 0)),  # multi-device code path (two host threads, one GPU)
])
def test_pipeline_equals_resident_batch(cfg, count, cap, its, devices):
    wl = workloads.CONFIGS[cfg]().strided(count)
    record_from = its - 2
    pool, plain, snaps = plain_run(wl, its, record_from)
    d = wl.model.dims()
    chunks = []

    def on_chunk(start, n, rec):
        chunks.append((start, n, rec))

    td, y, acc, oc = pkg.solve_pool(pool, wl.model, pkg.SolverConfig(wl.algorithm, wl.dt), cap, its,
                                    record_from=record_from, record_mask=0x1B, on_chunk=on_chunk,
                                    devices=devices)
    assert np.array_equal(td.view(np.uint64), plain["td"].view(np.uint64))
    assert np.array_equal(y.view(np.uint64), plain["y"].view(np.uint64))
    assert np.array_equal(acc.view(np.uint64), plain["acc"].view(np.uint64))
    assert np.array_equal(outcome_bytes(oc), outcome_bytes(plain["outcomes"]))
    # chunks tile the pool; recorded snapshots equal the resident run's sink view
    starts = sorted((s, n) for s, n, _ in chunks)
    assert starts[0][0] == 0 and sum(n for _, n in starts) == wl.n
    for s, n, rec in chunks:
        for r, (sy, sa, so) in enumerate(snaps):
            got_y = rec["state"].reshape(-1, d.system_dim, n)[r]
            want_y = sy.reshape(d.system_dim, wl.n)[:, s:s + n]
            assert np.array_equal(got_y, want_y)
            got_o = rec["outcomes"].reshape(-1, n)[r]
            assert np.array_equal(outcome_bytes(got_o), outcome_bytes(so[s:s + n]))


def test_persistent_pipeline_reuse():
    """odegpu_pipeline_* keeps its batches/staging across runs: two different
    pools, then the first again, reproduce the one-shot solve_pool bitwise."""
    a = workloads.cfg4().strided(2000)
    b = workloads.cfg4().subset(slice(5000, 6500))
    pools = [pkg.ProblemPool.from_arrays(*w.arrays()) for w in (a, b)]
    cfg = pkg.SolverConfig(a.algorithm, a.dt)
    want = [pkg.solve_pool(p, a.model, cfg, 600, 2) for p in pools]
    pipe = pkg.api.Pipeline(a.model, 600)
    recs = []
    for i in (0, 1, 0):
        got = pipe.run(pools[i], cfg, 2, record_from=1, record_mask=pkg.api.RECORD_STATE,
                       on_chunk=lambda s, n, r: recs.append((s, n)))
        for g, w in zip(got, want[i]):
            assert np.array_equal(np.ascontiguousarray(g).view(np.uint8), np.ascontiguousarray(w).view(np.uint8))
    assert sum(n for _, n in recs) == 2000 + 1500 + 2000
    pipe.close()


def test_pipeline_reports_bad_time_domain():
    wl = workloads.cfg2().strided(600)
    td, y, p, acc = wl.arrays()
    td[wl.n + 450] = -1.0  # t1 < t0 for system 450 (chunk 1, batch index 50)
    pool = pkg.ProblemPool.from_arrays(td, y, p, acc)
    with pytest.raises(pkg.InvalidArgument, match="system 50 has t1 < t0"):
        pkg.solve_pool(pool, wl.model, pkg.SolverConfig(wl.algorithm, wl.dt), 400, 1)


def test_batch_copy_restores_a_pristine_batch():
    wl = workloads.cfg3().strided(512)
    td, y, p, acc = wl.arrays()
    pool = pkg.ProblemPool.from_arrays(td, y, p, acc)
    dims = pkg.make_batch_dims(wl.n, wl.model.dims())
    pristine, work = pkg.SolverBatch(dims), pkg.SolverBatch(dims)
    pkg.linear_set(pristine, pool, pkg.LinearCopySpec(0, 0, wl.n))
    cfg = pkg.SolverConfig(wl.algorithm, wl.dt)
    results = []
    for _ in range(2):
        pkg.batch_copy(work, pristine)
        pkg.solve(work, wl.model, cfg)
        results.append(work.state())
    assert np.array_equal(results[0], results[1])
    assert np.array_equal(pristine.state(), y)
