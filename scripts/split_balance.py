"""How evenly the multi-GPU splits divide the work:
per-system trial steps of one solve of each BASELINE grid at full size
(iteration 1 for the in-place configs, as the bench times them), replayed
through (a) contiguous equal-count slices (odegpu_slice), (b) bench.py's
block-cyclic 4096-system blocks per rank, (c) odegpu_solve_pool_multi's
shared chunk queue (list scheduling of pool-order chunks onto devices as
they free up). Reports max/mean work per device for 2, 4, 8 devices.
    python scripts/split_balance.py > profiles/.../split_balance.jsonl"""
import heapq
import json
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1810_03931_b200 as pkg  # noqa: E402
from paper_1810_03931_b200 import workloads  # noqa: E402

BLOCK = 4096


def costs(name):
    wl = workloads.cfg5(24) if name == "cfg5" else workloads.CONFIGS[name]()
    td, y, p, acc = wl.arrays()
    pool = pkg.ProblemPool.from_arrays(td, y, p, acc)
    b = pkg.SolverBatch(pkg.make_batch_dims(wl.n, wl.model.dims()))
    pkg.linear_set(b, pool, pkg.LinearCopySpec(0, 0, wl.n))
    cfg = pkg.SolverConfig(wl.algorithm, wl.dt)
    if name in ("cfg3", "cfg4", "cfg5"):
        pkg.solve(b, wl.model, cfg)  # iteration 0; the bench times the iterations after it
    pkg.solve(b, wl.model, cfg)
    o = b.outcomes()
    c = (o["accepted_steps"] + o["rejected_steps"]).astype(np.float64)
    b.close()
    return wl.n, c


def contiguous(c, k):
    n = c.size
    base, extra = divmod(n, k)
    out, lo = [], 0
    for r in range(k):
        hi = lo + base + (1 if r < extra else 0)
        out.append(c[lo:hi].sum())
        lo = hi
    return np.array(out)


def cyclic(c, k, block=BLOCK):
    nb = -(-c.size // block)
    per_block = np.add.reduceat(c, np.arange(0, c.size, block))
    return np.array([per_block[r:nb:k].sum() for r in range(k)])


def rotated_owner(nb, k):
    """bench.py's block owners: each round of k consecutive blocks is dealt
    to the k ranks rotated by a hashed offset, so every rank gets the same
    number of blocks and no rank follows a fixed column of the grid."""
    b = np.arange(nb, dtype=np.uint64)
    rnd = b // np.uint64(k)
    off = ((rnd * np.uint64(0x9E3779B1)) >> np.uint64(11)) % np.uint64(k)
    return ((b + off) % np.uint64(k)).astype(np.int64)


def rotated(c, k, block):
    per_block = np.add.reduceat(c, np.arange(0, c.size, block))
    own = rotated_owner(per_block.size, k)
    return np.array([per_block[own == r].sum() for r in range(k)])


def queue(c, k, chunks_total=64):
    cap = -(-c.size // chunks_total)
    per_chunk = np.add.reduceat(c, np.arange(0, c.size, cap))
    heap = [(0.0, d) for d in range(k)]
    load = np.zeros(k)
    for w in per_chunk:  # pool order; the device that frees up first claims the next chunk
        t, d = heapq.heappop(heap)
        load[d] = t + w
        heapq.heappush(heap, (t + w, d))
    return load


for name in sys.argv[1:] or ["cfg2", "cfg3", "cfg4", "cfg5"]:
    n, c = costs(name)
    row = {"config": name, "systems": n, "trial_steps": float(c.sum())}
    for k in (2, 4, 8):
        for split, f in (("contiguous", contiguous), ("block_cyclic_4096", cyclic),
                         ("block_cyclic_1024", lambda c, k: cyclic(c, k, 1024)),
                         ("block_cyclic_256", lambda c, k: cyclic(c, k, 256)), ("chunk_queue_64", queue),
                         ("chunk_queue_256", lambda c, k: queue(c, k, 256)),
                         ("rotated_1024", lambda c, k: rotated(c, k, 1024)),
                         ("rotated_512", lambda c, k: rotated(c, k, 512)),
                         ("rotated_4096", lambda c, k: rotated(c, k, 4096))):
            w = f(c, k)
            row[f"{split}_{k}"] = round(float(w.max() / w.mean()), 4)
    print(json.dumps(row), flush=True)
