"""World-size-2 gloo test of the multi-GPU host logic on CPU.

Systems are independent, so the multi-GPU path has no data-path collective:
each rank owns a share of the pool and the results are gathered on the host.
Here each rank integrates its share with the C oracle standing in for its
device (no GPU here), the shares are all-gathered over gloo and must
reproduce the single-process run bitwise — for the contiguous odegpu_slice
split and for bench.py's block-cyclic strong-scaling split.
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
        # bench.py's strong-scaling split: block-cyclic blocks of bench.BLOCK
        import bench

        wl2 = workloads.cfg4().strided(3 * bench.BLOCK + 77)
        idx = bench.owned_indices(wl2.n, rank, world, "cyclic")
        r2 = pyoracle.solve_workload("port", wl2.subset(idx), 1)
        cyc = [None] * world
        dist.all_gather_object(cyc, (idx, r2["y"], r2["outcomes"]["accepted_steps"]))
        if rank == 0:
            out_q.put((gathered, cyc))
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
    gathered, cyc = q.get(timeout=240)
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

    # block-cyclic: the ranks' shares partition the pool and reassemble the
    # single-process run bitwise
    import bench

    wl2 = workloads.cfg4().strided(3 * bench.BLOCK + 77)
    full2 = pyoracle.solve_workload("port", wl2, 1)
    owner = np.full(wl2.n, -1)
    y2 = np.empty((dim, wl2.n))
    s2 = np.empty(wl2.n, dtype=np.int64)
    for r, (idx, ys, st) in enumerate(cyc):
        assert np.all(owner[idx] == -1)
        owner[idx] = r
        y2[:, idx] = ys.reshape(dim, idx.size)
        s2[idx] = st
    assert np.all(owner >= 0)
    assert np.array_equal(y2.reshape(-1).view(np.uint64), full2["y"].view(np.uint64))
    assert np.array_equal(s2, full2["outcomes"]["accepted_steps"])


def test_block_owner_deals_equal_shares_without_grid_resonance():
    """bench.py's strong-scaling owners: every round of `world` blocks is a
    permutation of the ranks (equal block counts), and the rotation breaks
    the fixed rank-to-column pattern of plain block-cyclic ownership."""
    import bench

    for world in (2, 3, 4, 8):
        own = bench.block_owner(1000 * world + 5, world)
        for r0 in range(0, 1000 * world, world):
            assert sorted(own[r0:r0 + world]) == list(range(world))
        # blocks 4 apart (one 4096-wide grid row of 1024-blocks) do not all
        # land on one rank, as they would with own = b % world for world = 4, 8
        row_start = own[0::4][:200]
        assert len(set(row_start.tolist())) == world
