"""Streaming pool pipeline (odegpu_pipeline_mode STREAMING, csrc/pipeline.cu
run_streaming): the pool lands chunk by chunk while ONE persistent solve
kernel runs over it, gated per chunk on device counters. Every system's
arithmetic depends only on its own data (solve.hpp:57-59), so the results
must be bitwise those of a resident batch and of the chunked pipeline, for
any stream chunk size, fused iterations, in-place write-back and systems the
certified pass defers to the general-trig pass."""
import numpy as np
import pytest

import paper_1810_03931_b200 as pkg
from paper_1810_03931_b200 import abi, workloads
from paper_1810_03931_b200.api import PIPELINE_CHUNKED, PIPELINE_STREAMING, Pipeline, pinned

pytestmark = pytest.mark.gpu


def outcome_bytes(o):
    raw = np.ascontiguousarray(o).view(np.uint8).reshape(-1, 56)
    return raw[:, [i for i in range(56) if not 9 <= i < 16]]


def resident(wl, iterations, td, y, p, acc):
    pool = pkg.ProblemPool.from_arrays(td, y, p, acc)
    b = pkg.SolverBatch(pkg.make_batch_dims(wl.n, wl.model.dims()))
    pkg.linear_set(b, pool, pkg.LinearCopySpec(0, 0, wl.n))
    pkg.solve_iteratively(b, wl.model, pkg.SolverConfig(wl.algorithm, wl.dt), iterations)
    return b.time_domain(), b.state(), b.accessories(), b.outcomes()


def pinned_outs(wl):
    d = wl.model.dims()
    n = wl.n
    return (pinned(np.zeros(2 * n)), pinned(np.zeros(d.system_dim * n)), pinned(np.zeros(max(d.accessory_count, 1) * n)),
            pinned(np.zeros(n, dtype=abi.OUTCOME_DTYPE)))


def assert_same(got, want, d):
    td, y, acc, oc = got
    assert np.array_equal(td.view(np.uint64), want[0].view(np.uint64))
    assert np.array_equal(y.view(np.uint64), want[1].view(np.uint64))
    if d.accessory_count:
        assert np.array_equal(acc[:want[2].size].view(np.uint64), want[2].view(np.uint64))
    assert np.array_equal(outcome_bytes(oc), outcome_bytes(want[3]))


@pytest.mark.parametrize("cfg,count,chunk", [
    ("cfg2", 5000, "96"), ("cfg2", 4097, ""), ("cfg3", 3000, "256"), ("cfg4", 3001, "160"), ("cfg1", 700, "64"),
])
def test_streaming_equals_resident_and_chunked(cfg, count, chunk, monkeypatch):
    if chunk:
        monkeypatch.setenv("ODEGPU_STREAM_CHUNK", chunk)
    wl = workloads.CONFIGS[cfg]().strided(count)
    td, y, p, acc = wl.arrays()
    want = resident(wl, 1, td, y, p, acc)
    pool = pkg.ProblemPool.from_arrays(td, y, p, acc).pin()
    cfgc = pkg.SolverConfig(wl.algorithm, wl.dt)
    d = wl.model.dims()
    stream = Pipeline(wl.model, 1024, mode=PIPELINE_STREAMING)
    outs = pinned_outs(wl)
    stream.run(pool, cfgc, 1, out_arrays=outs)
    assert stream.last_mode() == PIPELINE_STREAMING
    assert_same(outs, want, d)
    chunked = Pipeline(wl.model, 1024, mode=PIPELINE_CHUNKED)
    outs2 = pinned_outs(wl)
    chunked.run(pool, cfgc, 1, out_arrays=outs2)
    assert chunked.last_mode() == PIPELINE_CHUNKED
    assert_same(outs2, want, d)
    # a second streaming run through the same pipeline (state reset per run)
    outs3 = pinned_outs(wl)
    stream.run(pool, cfgc, 1, out_arrays=outs3)
    assert_same(outs3, want, d)
    stream.close()
    chunked.close()


@pytest.mark.parametrize("cfg,count,its", [("cfg3", 2048, 3), ("cfg4", 2500, 2), ("cfg1", 512, 4)])
def test_streaming_in_place_fused_iterations(cfg, count, its, monkeypatch):
    """In place (out arrays = the pool's own arrays) with fused iterations:
    the end points of iteration `its`, as a resident solve_iteratively."""
    monkeypatch.setenv("ODEGPU_STREAM_CHUNK", "128")
    wl = workloads.CONFIGS[cfg]().strided(count)
    td, y, p, acc = wl.arrays()
    want = resident(wl, its, td, y, p, acc)
    pool = pkg.ProblemPool.from_arrays(td, y, p, acc).pin()
    oc = pinned(np.zeros(wl.n, dtype=abi.OUTCOME_DTYPE))
    pipe = Pipeline(wl.model, 700, mode=PIPELINE_STREAMING)
    pipe.run(pool, pkg.SolverConfig(wl.algorithm, wl.dt), its,
             out_arrays=(pool._td, pool._state, pool._acc if wl.model.dims().accessory_count else None, oc))
    assert pipe.last_mode() == PIPELINE_STREAMING
    assert_same((pool._td, pool._state, pool._acc, oc), want, wl.model.dims())
    pipe.close()


def test_streaming_integrates_systems_beyond_the_trig_certificate(monkeypatch):
    """The streaming pass takes the general trig path (the certificate would
    need every system before the launch): systems whose trig arguments need
    Payne-Hanek reduction are integrated like the rest — bitwise the
    resident batch (whose certificate then fails for the whole batch)."""
    monkeypatch.setenv("ODEGPU_STREAM_CHUNK", "64")
    wl = workloads.cfg2().strided(1000)
    td, y, p, acc = wl.arrays()
    n = wl.n
    for i in (3, 400, 401, 999):  # omega * t beyond 2^31: Payne-Hanek territory
        td[i] += 3.0e9
        td[n + i] += 3.0e9
    want = resident(wl, 1, td, y, p, acc)
    pool = pkg.ProblemPool.from_arrays(td, y, p, acc).pin()
    outs = pinned_outs(wl)
    pipe = Pipeline(wl.model, 256, mode=PIPELINE_STREAMING)
    pipe.run(pool, pkg.SolverConfig(wl.algorithm, wl.dt), 1, out_arrays=outs)
    assert_same(outs, want, wl.model.dims())
    pipe.close()


def test_streaming_reports_bad_time_domain_like_chunked():
    wl = workloads.cfg2().strided(600)
    td, y, p, acc = wl.arrays()
    td[wl.n + 450] = -1.0  # t1 < t0 for system 450 (chunk 1 of 400, batch index 50)
    td[wl.n + 520] = -1.0
    pool = pkg.ProblemPool.from_arrays(td, y, p, acc).pin()
    cfgc = pkg.SolverConfig(wl.algorithm, wl.dt)
    for mode in (PIPELINE_STREAMING, PIPELINE_CHUNKED):
        pipe = Pipeline(wl.model, 400, mode=mode)
        with pytest.raises(pkg.InvalidArgument, match="system 50 has t1 < t0"):
            pipe.run(pool, cfgc, 1, out_arrays=pinned_outs(wl))
        pipe.close()
    # the pipeline stays usable after the error
    td[wl.n + 450] = td[wl.n + 449]
    td[wl.n + 520] = td[wl.n + 519]
    pool = pkg.ProblemPool.from_arrays(td, y, p, acc).pin()
    pipe = Pipeline(wl.model, 400, mode=PIPELINE_STREAMING)
    outs = pinned_outs(wl)
    pipe.run(pool, cfgc, 1, out_arrays=outs)
    assert_same(outs, resident(wl, 1, td, y, p, acc), wl.model.dims())
    pipe.close()


def test_streaming_needs_page_locked_arrays():
    wl = workloads.cfg4().strided(300)
    pool = pkg.ProblemPool.from_arrays(*wl.arrays())  # pageable
    pipe = Pipeline(wl.model, 128, mode=PIPELINE_STREAMING)
    with pytest.raises(pkg.Unsupported, match="page-locked"):
        pipe.run(pool, pkg.SolverConfig(wl.algorithm, wl.dt), 1)
    pipe.set_mode(pkg.api.PIPELINE_AUTO)  # AUTO runs the chunked slots
    pipe.run(pool, pkg.SolverConfig(wl.algorithm, wl.dt), 1)
    assert pipe.last_mode() == PIPELINE_CHUNKED
    pipe.close()


def test_auto_mode_runs_the_chunked_slots():
    """AUTO (the default) runs the chunked slots; STREAMING is opt-in."""
    wl = workloads.CONFIGS["cfg2"]().strided(300)
    pool = pkg.ProblemPool.from_arrays(*wl.arrays()).pin()
    pipe = Pipeline(wl.model, 128)
    pipe.run(pool, pkg.SolverConfig(wl.algorithm, wl.dt), 1, out_arrays=pinned_outs(wl))
    assert pipe.last_mode() == PIPELINE_CHUNKED
    pipe.close()
