"""World-size-2 gloo test of the multi-GPU host logic on CPU.

Systems are independent, so the multi-GPU path has no data-path collective:
each rank owns the contiguous slice odegpu_slice(N, world, rank) and the
results are gathered on the host. Here each rank integrates its slice with
the C oracle (no GPU needed), the slices are all-gathered over gloo and must
reproduce the single-process run bitwise; bench.py's weak-scaling workload
split is checked the same way.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_q):
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    sys.path.insert(0, str(root))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1810_03931_b200 as pkg
        from oracle import pyoracle
        from paper_1810_03931_b200 import workloads

        wl = workloads.cfg4().strided(600)
        b, e = pkg.slice_range(wl.n, world, rank)
        mine = wl.subset(slice(b, e))
        r = pyoracle.solve_workload("port", mine, 2)
        gathered = [None] * world
        dist.all_gather_object(gathered, (b, e, r["y"], r["outcomes"]["accepted_steps"]))
        # bench.py weak-scaling split of the cfg2 grid
        import bench

        wl2 = bench.make_workload("cfg2", rank, world)
        rows = [None] * world
        dist.all_gather_object(rows, wl2.p[0][::1024].copy())
        if rank == 0:
            out_q.put((gathered, rows))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_slices_reproduce_single_process_run():
    import paper_1810_03931_b200 as pkg
    from oracle import pyoracle
    from paper_1810_03931_b200 import workloads

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    gathered, rows = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0

    wl = workloads.cfg4().strided(600)
    full = pyoracle.solve_workload("port", wl, 2)
    n, dim = wl.n, wl.model.dims().system_dim
    y = np.empty((dim, n))
    steps = np.empty(n, dtype=np.int64)
    covered = 0
    for b, e, ys, acc_steps in gathered:
        y[:, b:e] = ys.reshape(dim, e - b)
        steps[b:e] = acc_steps
        covered += e - b
    assert covered == n
    assert np.array_equal(y.reshape(-1).view(np.uint64), full["y"].view(np.uint64))
    assert np.array_equal(steps, full["outcomes"]["accepted_steps"])
    assert pkg.slice_range(600, 2, 0) == (0, 300) and pkg.slice_range(601, 2, 1) == (301, 601)

    # weak scaling: rank r owns k-rows [r*1024, (r+1)*1024) of a 2048 x 1024 grid
    k_all = np.concatenate(rows)
    assert np.array_equal(k_all, workloads.param_range(0.2, 0.3, 2048))
