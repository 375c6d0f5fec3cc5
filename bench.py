#!/usr/bin/env python
"""Benchmark of the ensemble-solve hot path (BASELINE.json metric: FP64 RK
steps/s and systems/s, % of FP64 peak, vs the host CPU).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg5 --log2n 24]
    python bench.py --impl reference ...   # the reference CPU solver arm

Default workload: BASELINE.json configs[4] at its largest single-GPU size —
the Keller-Miksis scaling pool of 2^24 systems (4096 PA1 x 4096 f1, RKCK45
tol 1e-10, BubbleCollapseSystem), iterated IN PLACE the way the reference's
run_bubble_scan drives it (src/scan.cpp:247-329 -> solve_iteratively,
solve.hpp:133-142): every step is one solve() over the whole pool that
continues from the previous step's end point (one collapse per system).

* value: trial steps (accepted + rejected, counted on the device) per second,
  pool resident in HBM. Timed with ONE pair of CUDA events on the batch stream
  around all K steps (plus the per-step device outcome tally), bracketed by a
  barrier + synchronize; max over ranks. The pool (3.3 GB at 2^24) is larger
  than L2, so no flush is needed between steps.
* fetch order (AUTO policy): Keller-Miksis pools in index order (the cost
  order measured even at 2^24 and doubled DRAM traffic), the valve longest
  first by each system's cost in the PREVIOUS iteration — information a real
  scan has. cfg2 cannot iterate in place (the reference's secant Zeno loop,
  DESIGN.md §4): every step restarts from the initial conditions and runs in
  natural order.
* e2e: the same metric through the C ABI with host (pinned) buffers — the
  chunked pool pipeline (odegpu_pipeline_run): per step H2D of the pool, one
  in-place iteration, D2H of the end points and outcome records into the
  host pool, wall clock.
* roofline: FP64-pipe instructions per trial step (SURVEY.md §8d algorithmic
  count) x device-counted trial steps / solve-kernel time vs the DFMA
  microbenchmark peak measured in the same run.
* cpu_baseline: the reference solver (oracle/_ref, compiled from the
  reference's own sources) on this box's host cores, bounded sample.

Multi-GPU (torchrun, or `--gpus N` which relaunches itself under torchrun):
STRONG scaling of the same fixed pool. Rank r owns the 1024-system blocks
block_owner() deals it (rounds of N blocks, rotated by a hashed offset: every
rank samples the whole grid, so the per-rank work is balanced without any
exchange — 8-way max/mean <= 1.0024 on the measured costs); no collective on
the data path — the barrier and MAX/SUM all-reduces of the timing are the
only communication.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import paper_1810_03931_b200 as pkg  # noqa: E402
from paper_1810_03931_b200 import abi, workloads  # noqa: E402

METRIC = "FP64 RK trial steps/s"
UNIT = "steps/s"
BLOCK = 1024  # ownership granule of the multi-rank split (block_owner)


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg5", choices=sorted(workloads.CONFIGS) + ["cfg5"])
    ap.add_argument("--log2n", type=int, default=24, help="cfg5: Keller-Miksis pool of 2^log2n systems")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--e2e-chunks", type=int, default=0, help="pipeline chunks for e2e (0 = by pool size)")
    ap.add_argument("--cpu-sample", type=int, default=0, help="systems in the CPU sample (0 = auto)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-natural", action="store_true", help="skip the natural-order comparison solve")
    ap.add_argument("--partition", default="cyclic", choices=["cyclic", "contiguous"],
                    help="multi-rank split: block-cyclic (balanced) or contiguous slices (odegpu_slice)")
    ap.add_argument("--allow-shared-gpu", action="store_true",
                    help="let more ranks than GPUs share devices (tests only; the rate is then shared too)")
    return ap.parse_args(argv)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def relaunch_under_torchrun(args) -> int:
    """`python bench.py --gpus N` without torchrun: one process per GPU."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve())] + sys.argv[1:]
    return subprocess.call(cmd)


def full_workload(args):
    return workloads.cfg5(args.log2n) if args.config == "cfg5" else workloads.CONFIGS[args.config]()


def workload_name(args, wl):
    return f"cfg5_keller_miksis_2^{args.log2n}" if args.config == "cfg5" else wl.name


def owned_indices(n: int, rank: int, world: int, partition: str) -> np.ndarray:
    """Systems rank `rank` integrates: block-cyclic blocks of BLOCK, or the
    contiguous odegpu_slice share."""
    if world == 1:
        return np.arange(n)
    if partition == "contiguous":
        lo, hi = pkg.slice_range(n, world, rank)
        return np.arange(lo, hi)
    blocks = np.nonzero(block_owner(-(-n // BLOCK), world) == rank)[0]
    idx = (blocks[:, None] * BLOCK + np.arange(BLOCK)[None, :]).reshape(-1)
    return idx[idx < n]


def block_owner(n_blocks: int, world: int) -> np.ndarray:
    """Owner rank of each BLOCK-system block: every round of `world`
    consecutive blocks is dealt to the ranks rotated by a hashed offset, so
    each rank owns the same number of blocks and no rank follows a fixed
    column of a parameter grid (plain block-cyclic blocks of 1024 resonate
    with cfg5's 4096-wide rows: 8-way max/mean work 1.34). Replayed with the
    measured per-system costs (scripts/split_balance.py,
    profiles/r02z/split_balance.jsonl), 8-way max/mean work is <= 1.0024 on
    cfg2-cfg5 (contiguous slices: 1.45 on cfg4)."""
    b = np.arange(n_blocks, dtype=np.uint64)
    off = (((b // np.uint64(world)) * np.uint64(0x9E3779B1)) >> np.uint64(11)) % np.uint64(world)
    return ((b + off) % np.uint64(world)).astype(np.int64)


def keller_miksis(wl) -> bool:
    """Keller-Miksis pools take their systems in index order under AUTO."""
    return wl.model.to_c().id in (abi.MODEL_KELLER_MIKSIS, abi.MODEL_BUBBLE_COLLAPSE)


def in_place(config: str) -> bool:
    """cfg2 restarts every step (the reference's own solver hits a Zeno loop
    when its grid is iterated in place); the rest iterate."""
    return config != "cfg2"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region (pynvml)."""

    def __init__(self, device: int):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # pragma: no cover - no NVML
            self._nv = None
            self.error = str(e)

    _NAMES = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self._nv.nvmlDeviceGetClockInfo(self._h, self._nv.NVML_CLOCK_SM))
                r = self._nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for bit, name in self._NAMES.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.05)

    def __enter__(self):
        if self._nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._nv:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def load_traffic(name: str):
    """DRAM bytes per solve-kernel launch from the committed ncu summary."""
    p = ROOT / "profiles" / "ncu_summary.json"
    if not p.exists():
        return None
    try:
        d = json.loads(p.read_text())
        return d.get("traffic_bytes_per_launch", {}).get(name)
    except Exception:
        return None


def host_info() -> dict:
    """CPU model, physical cores and the threads this process may use (lscpu)."""
    info = {"threads_available": len(os.sched_getaffinity(0))}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        kv = {}
        for line in out.splitlines():
            if ":" in line:
                k, v = line.split(":", 1)
                kv[k.strip()] = v.strip()
        info["cpu_model"] = kv.get("Model name")
        cps, sockets = kv.get("Core(s) per socket"), kv.get("Socket(s)")
        if cps and sockets and cps.isdigit() and sockets.isdigit():
            info["physical_cores"] = int(cps) * int(sockets)
        info["logical_cpus"] = int(kv["CPU(s)"]) if kv.get("CPU(s)", "").isdigit() else None
    except Exception:
        pass
    return info


def reference_rate(wl, sample: int, warmup: int, steps: int, workers: int, in_place_iter: bool):
    """The reference solver (oracle/_ref) on a strided sample of the workload,
    stepped exactly like the GPU arm: `warmup` untimed iterations, then
    `steps` timed ones (in place, or each from the initial conditions)."""
    from oracle import pyoracle

    sub = wl.strided(sample)
    td, y, p, acc = sub.arrays()
    oc = abi.empty_outcomes(sub.n)
    kw = dict(algorithm=sub.algorithm, dt=sub.dt, iterations=1, workers=workers, outcomes=oc)
    for _ in range(warmup):
        if not in_place_iter:
            td, y, p, acc = sub.arrays()
            oc[:] = abi.empty_outcomes(sub.n)
        pyoracle.solve("reference", sub.model, td, y, p, acc, **kw)
    total_steps, total_s = 0, 0.0
    for _ in range(steps):
        if not in_place_iter:
            td, y, p, acc = sub.arrays()
            oc[:] = abi.empty_outcomes(sub.n)
        _, secs, _ = pyoracle.solve("reference", sub.model, td, y, p, acc, **kw)
        total_steps += int(oc["accepted_steps"].sum() + oc["rejected_steps"].sum())
        total_s += secs
    return total_steps / total_s, sub.n * steps / total_s, sub.n, total_s


def cpu_baseline(wl, args, sample: int):
    """Reference solver on all host threads (bounded sample) plus a 1-thread
    figure on a smaller sample, with the CPU model and core counts."""
    from oracle import pyoracle

    if not pyoracle.available("reference"):
        return None
    info = host_info()
    threads = info["threads_available"]
    ip = in_place(args.config)
    rate, sys_rate, n_s, secs = reference_rate(wl, sample, 1, 2, threads, ip)
    rate1, _, n_1, secs1 = reference_rate(wl, max(sample // max(threads, 1), 256), 1, 1, 1, ip)
    return {"value": rate, "unit": UNIT, "cores": threads, "kind": "reference",
            "sample": f"{n_s} of {wl.n} systems (evenly strided), 1 untimed + 2 timed "
                      f"{'in-place iterations' if ip else 'solves from the initial conditions'}, "
                      f"{secs:.2f} s timed, reference solve() with worker_count={threads}",
            "systems_per_s": sys_rate,
            "one_thread": {"value": rate1, "sample": f"{n_1} systems, 1 timed iteration, {secs1:.2f} s"},
            "host": info}


def run_reference_arm(args, rank, world):
    """--impl reference: the reference CPU solver on this box's host cores,
    same metric and config as our arm (bounded sample per step)."""
    if rank != 0:
        return
    from oracle import pyoracle

    wl = full_workload(args)
    if not pyoracle.available("reference"):
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libodref.so not built"}))
        return
    info = host_info()
    threads = info["threads_available"]
    sample = args.cpu_sample or {"cfg1": 46080, "cfg2": 1 << 19, "cfg3": 1 << 16, "cfg4": 1 << 17,
                                 "cfg5": 1 << 16}[args.config]
    ip = in_place(args.config)
    value, sys_rate, n_s, total_s = reference_rate(wl, sample, args.warmup, args.steps, threads, ip)
    desc = (f"{n_s} of {wl.n} systems (evenly strided) per step, "
            f"{'iterated in place' if ip else 'each step from the initial conditions'}, "
            f"reference solve() on {threads} threads")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total_s / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_name(args, wl), "description": wl.description, "sample": desc},
        "systems_per_s": sys_rate,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference", "sample": desc,
                         "host": info},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


_T0 = time.time()


def log(msg: str):
    print(f"[bench +{time.time() - _T0:7.1f}s] {msg}", file=sys.stderr, flush=True)


def pinned_like(torch, a: np.ndarray) -> np.ndarray:
    """A page-locked copy of `a` (numpy view of pinned torch storage)."""
    buf = torch.empty(max(a.size, 1), dtype=torch.float64, pin_memory=True).numpy()[: a.size]
    buf[:] = a
    return buf


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_under_torchrun(args))
    shared = False
    if world > 1:
        import torch
        import torch.distributed as dist

        shared = torch.cuda.device_count() < world
        if shared and args.impl == "ours" and not args.allow_shared_gpu:
            if rank == 0:
                print(json.dumps({"error": f"{world} ranks but {torch.cuda.device_count()} visible GPUs "
                                           "(pass --allow-shared-gpu to share devices in a test)"}))
            sys.exit(2)
        dist.init_process_group("nccl" if args.impl == "ours" and not shared else "gloo")
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()
        return

    import torch

    device = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(device)
    red_dev = f"cuda:{device}" if world > 1 and torch.distributed.get_backend() == "nccl" else "cpu"
    log(f"torch ready, rank {rank}/{world} on cuda:{device}")

    def allreduce(vals, op):
        if world == 1:
            return vals
        import torch.distributed as dist

        t = torch.tensor(vals, dtype=torch.float64, device=red_dev)
        dist.all_reduce(t, op=op)
        return [float(v) for v in t.tolist()]

    full = full_workload(args)
    mine = owned_indices(full.n, rank, world, args.partition)
    wl = full if world == 1 else full.subset(mine)
    n = wl.n
    ip = in_place(args.config)
    td, y, p, acc = wl.arrays()
    pool = pkg.ProblemPool.from_arrays(td, y, p, acc)
    batch = pkg.SolverBatch(pkg.make_batch_dims(n, wl.model.dims()), device=device)
    stream = torch.cuda.Stream(device=device)
    batch.set_stream(stream.cuda_stream)
    cfg = pkg.SolverConfig(wl.algorithm, wl.dt)
    pkg.linear_set(batch, pool, pkg.LinearCopySpec(0, 0, n))
    pristine = None
    if not ip:  # cfg2: every step from the initial conditions, natural order
        pristine = pkg.SolverBatch(pkg.make_batch_dims(n, wl.model.dims()), device=device)
        pkg.batch_copy(pristine, batch)
        batch.set_fetch_order(abi.FETCH_NATURAL)

    log(f"{wl.name}: {n} of {full.n} systems resident on this rank")
    peak_lane, _ = pkg.dfma_peak(device)
    log(f"DFMA peak {peak_lane:.4e} lane-DFMA/s")

    if ip:  # the scan's first (transient) iterations, fused like the timed ones
        pkg.solve_iteratively(batch, wl.model, cfg, args.warmup)
    else:
        for _ in range(args.warmup):
            pkg.batch_copy(batch, pristine)
            pkg.solve(batch, wl.model, cfg)

    # ---------------- timed region (device-resident pool)
    # in place: ONE solve_iteratively(K) call without a sink — the transient
    # iterations of a scan; the built-in models fuse them (each lane solves
    # its system K times in a row in one launch, hooks.hpp
    # kFusableIterations). cfg2: K solves from the initial conditions.
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    batch.trial_steps(reset=True)
    launches0 = batch.launch_count()
    kern_ms, certified = [], False
    e_start = torch.cuda.Event(enable_timing=True)
    e_end = torch.cuda.Event(enable_timing=True)
    with ClockSampler(device) as clocks:
        w0 = time.perf_counter()
        e_start.record(stream)
        if ip:
            pkg.solve_iteratively(batch, wl.model, cfg, args.steps)
            kern_ms.append(batch.last_kernel_ms())
        else:
            for _ in range(args.steps):
                pkg.batch_copy(batch, pristine)  # outside the kernel-time events (inside the span)
                pkg.solve(batch, wl.model, cfg)
                kern_ms.append(batch.last_kernel_ms())
        e_end.record(stream)
        e_end.synchronize()
        wall = time.perf_counter() - w0
        certified = batch.trig_certified()
    torch.cuda.synchronize()
    launches = batch.launch_count() - launches0
    steps_total = batch.trial_steps()
    max_trial = batch.diagnostics()["max_trial_steps"]  # last iteration, outside the timing
    span_s = e_start.elapsed_time(e_end) / 1e3
    # solve-kernel time: the fused launch (in place), else the sum of the K
    # launches; a model that could not fuse ran K launches: only the last
    # one's events exist, so the span stands in for the kernel time
    kernel_s = sum(kern_ms) / 1e3
    if ip and kernel_s < 0.5 * span_s:
        kernel_s = span_s
    span_s, kernel_s, wall = allreduce([span_s, kernel_s, wall], torch.distributed.ReduceOp.MAX if world > 1 else None)
    steps_total, sys_total = allreduce([steps_total, n * args.steps],
                                       torch.distributed.ReduceOp.SUM if world > 1 else None)
    steps_total, sys_total = int(steps_total), int(sys_total)
    # Ranks sharing one GPU (--allow-shared-gpu, tests only) are time-sliced
    # by the driver: each rank's CUDA-event span covers only its own slices,
    # so the max over ranks would claim their sum as parallel work. There
    # the region is the wall clock between the barriers, max over ranks.
    if shared:
        span_s = max(span_s, wall)
        kernel_s = span_s
    value = steps_total / span_s
    achieved = steps_total * wl.instr_per_step / kernel_s  # lane FP64-pipe instr/s (all ranks)
    peak_total = peak_lane * (min(world, torch.cuda.device_count()) if shared else world)
    log(f"timed region done: {steps_total} trial steps in {span_s:.4f} s (kernels {kernel_s:.4f} s)")

    # ---------------- the same iterations in natural fetch order (outside the
    # timed region): a snapshot of the pool is solved once ordered, once not
    natural = None
    if ip and wl.algorithm == abi.RKCK45 and not keller_miksis(wl) and not args.no_natural:
        k_nat = min(args.steps, 3)
        snap = pkg.SolverBatch(pkg.make_batch_dims(n, wl.model.dims()), device=device)
        pkg.batch_copy(snap, batch)
        pkg.solve_iteratively(batch, wl.model, cfg, k_nat)
        ordered_ms = batch.last_kernel_ms()
        pkg.batch_copy(batch, snap)
        batch.set_fetch_order(abi.FETCH_NATURAL)
        batch.trial_steps(reset=True)
        pkg.solve_iteratively(batch, wl.model, cfg, k_nat)
        natural_ms = batch.last_kernel_ms()
        st = batch.trial_steps()
        natural = {"iterations": k_nat, "ordered_kernel_ms": ordered_ms, "natural_kernel_ms": natural_ms,
                   "frac_natural_order": st * wl.instr_per_step / (natural_ms / 1e3) / peak_lane,
                   "frac_previous_iteration_order": st * wl.instr_per_step / (ordered_ms / 1e3) / peak_lane}
        snap.close()
    batch.close()
    if pristine is not None:
        pristine.close()

    # ---------------- e2e: through the C ABI with host buffers, per step
    h_td, h_y, h_p, h_a = (pinned_like(torch, a) for a in (td, y, p, acc))
    pin_pool = pkg.ProblemPool.from_arrays(td, y, p, acc)
    pin_pool._td, pin_pool._state, pin_pool._params, pin_pool._acc = h_td, h_y, h_p, h_a
    outc = torch.zeros(n * abi.OUTCOME_DTYPE.itemsize, dtype=torch.uint8, pin_memory=True).numpy().view(
        abi.OUTCOME_DTYPE)
    h2d = h_td.nbytes + h_y.nbytes + h_p.nbytes + h_a.nbytes
    # time domains a solve cannot change are not read back (hooks.hpp
    # kKeepsTimeDomain: the Duffing and valve models): in place the pipeline
    # skips them itself; restarted from the pool (cfg2) the result's time
    # domains are the pool's, so the out view leaves them out
    td_back = not wl.model.keeps_time_domain()
    d2h = (h_td.nbytes if td_back else 0) + h_y.nbytes + h_a.nbytes + outc.nbytes
    # chunks through the copy-in / kernels / copy-out pipeline (in place: end
    # points go back into the pool arrays). ~64 Ki systems per chunk, 2..8
    # chunks for the transfer-bound cheap models, up to 16 for Keller-Miksis
    # (scripts/e2e_chunks.py)
    n_chunks = args.e2e_chunks or int(min(max(round(n / 65536), 2), 16 if wl.instr_per_step > 500 else 8))
    cap = max(1, -(-n // n_chunks))
    pipe = pkg.api.Pipeline(wl.model, cap, device)
    outs = (h_td, h_y, h_a, outc) if ip else (pinned_like(torch, td) if td_back else None, pinned_like(torch, y),
                                              pinned_like(torch, acc), outc)
    pipe.run(pin_pool, cfg, 1, out_arrays=outs)  # warm-up (first touch of the staging)
    if world > 1:
        torch.distributed.barrier()
    # the timed region holds the product call alone (H2D, solve, D2H into the
    # host arrays); counting the trial steps of the result is bookkeeping of
    # this benchmark and happens outside it
    e2e_steps, e2e_s = 0, 0.0
    for _ in range(args.e2e_steps):
        t0 = time.perf_counter()
        pipe.run(pin_pool, cfg, 1, out_arrays=outs)
        e2e_s += time.perf_counter() - t0
        e2e_steps += int(outc["accepted_steps"].sum() + outc["rejected_steps"].sum())
    e2e_mode = pipe.last_mode()
    pipe.close()
    (e2e_s,) = allreduce([e2e_s], torch.distributed.ReduceOp.MAX if world > 1 else None)
    (e2e_steps,) = allreduce([e2e_steps], torch.distributed.ReduceOp.SUM if world > 1 else None)
    e2e_value = e2e_steps / e2e_s
    log(f"e2e done ({e2e_value:.4e} steps/s)")

    if rank != 0:
        if world > 1:
            torch.distributed.barrier()
            torch.distributed.destroy_process_group()
        return

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        sample = args.cpu_sample or {"cfg1": 46080, "cfg2": 1 << 19, "cfg3": 1 << 16, "cfg4": 1 << 17,
                                     "cfg5": 1 << 16}[args.config]
        log(f"CPU baseline on {sample} systems")
        cpu = cpu_baseline(full, args, sample)

    traffic = load_traffic(wl.name)
    per_launch_s = kernel_s / args.steps
    dims = wl.model.dims()
    hbm_bytes = n * 8 * (2 * 2 + 2 * dims.system_dim + dims.param_count + 2 * dims.accessory_count) + n * 49
    out = {
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": 1e3 * span_s / args.steps,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic",
        "config": {
            "workload": workload_name(args, wl),
            "description": full.description,
            "systems": full.n,
            "systems_per_gpu": n,
            "step": ("one in-place solve() iteration of the whole pool; the K timed steps are ONE "
                     "solve_iteratively(K) call without a sink (a scan's transient iterations), fused into one "
                     "kernel launch (one collapse / forcing period / section-to-section iteration per system "
                     "and step)") if ip else
                    "one solve() of the whole pool from its initial conditions (one forcing period)",
            "algorithm": "RK4" if wl.algorithm == abi.RK4 else "RKCK45",
            "l2": ("inputs larger than L2 (pool of %.2f GB resident in HBM), no flush" % (hbm_bytes / 1e9)),
            "parallelism": (f"dp{world}: rotated rounds of {BLOCK}-system blocks per rank" if args.partition == "cyclic"
                            else f"dp{world}: contiguous slices") if world > 1 else "single GPU",
            "timing": ("wall clock between barriers, max over ranks (ranks share a GPU)" if shared else
                       "CUDA events on each rank's batch stream, max over ranks"),
            "trig_path": "certified (branch-free, include/odegpu/trig.hpp)" if certified else "general",
            "fetch_order": ("longest first by each system's RK evaluations in the PREVIOUS iteration (AUTO "
                            "policy, what an in-place scan knows)") if ip and wl.algorithm == abi.RKCK45 and
                           not keller_miksis(wl) else
                           "natural (index order; AUTO for Keller-Miksis and fixed-step RK4, "
                           "csrc/models_keller_miksis.cu)",
            "natural_order": natural,
            "library": os.environ.get("ODEGPU_LIB") or ("parity" if os.environ.get("ODEGPU_BUILD") == "parity"
                                                         else "libodegpu.so (fast build)"),
        },
        "systems_per_s": sys_total / span_s,
        "trial_steps_per_system_step": steps_total / max(sys_total, 1),
        "max_trial_steps_one_system": max_trial,
        "gpu_launches": launches,
        "fused_iterations_per_launch": args.steps if ip else 1,
        "kernel_ms_per_step": 1e3 * per_launch_s,
        "wall_s_timed_region": wall,
        "roofline": {
            "bound": "fp64",
            "achieved": achieved / 1e9,
            "peak": peak_total / 1e9,
            "unit": "G lane-FP64-instr/s",
            "frac": achieved / peak_total,
            "traffic": traffic,
            "algorithmic": f"{wl.instr_per_step} FP64-pipe instructions per trial step (SURVEY.md §8d count, "
                           f"controller pow as the 13-instruction fifth root; DESIGN.md §3.1) x "
                           f"device-counted trial steps / solve-kernel time (CUDA events on the batch stream)",
            "peak_source": "DFMA microbenchmark in this run (odegpu_dfma_peak, 8 independent chains/thread); "
                           "MEASURED_PEAKS.json has no FP64 entry",
            "tflops_fp64": steps_total * wl.flops_per_step / kernel_s / 1e12,
            "hbm_gbs": hbm_bytes * world / per_launch_s / 1e9,
        },
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d) * world,
                "d2h_bytes_per_step": int(d2h) * world, "steps": args.e2e_steps,
                "mode": "streaming" if e2e_mode == pkg.api.PIPELINE_STREAMING else "chunked",
                "path": ("odegpu_pipeline_run over the pinned host pool, STREAMING mode: the pool lands chunk by "
                         "chunk (copy-in stream, device counter bumped per chunk) while ONE persistent solve kernel "
                         "runs over it; each chunk's end points and outcome records go back (copy-out stream) as "
                         "soon as its systems are counted done, "
                         if e2e_mode == pkg.api.PIPELINE_STREAMING else
                         f"odegpu_pipeline_run over the pinned host pool: {n_chunks} chunks per rank, H2D / "
                         "kernels / D2H of td, state, accessories and outcome records on separate streams, ")
                        + ("one in-place iteration per step (end points written back into the pool), "
                           if ip else "") + "wall clock, max over ranks"},
        "cpu_baseline": cpu,
        "clocks": clocks.summary(),
    }
    print(json.dumps(out))
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
