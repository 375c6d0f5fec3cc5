#!/usr/bin/env python
"""Benchmark of the ensemble-solve hot path (BASELINE.json metric: FP64 RK
steps/s and systems/s, % of FP64 peak, vs the host CPU).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2]
    python bench.py --impl reference ...   # the reference CPU solver arm

A "step" is one solve() over the whole batch (one solve_iteratively
iteration). Default workload: BASELINE.json configs[1] — Duffing RKCK45 with
the local-maximum EventFunction and event-time accessories on a 1024 x 1024
(damping x forcing) grid of 2^20 systems.

* value: trial steps (accepted + rejected, counted on the device) per second
  of device time with the batch resident in HBM; timed with CUDA events on the
  batch's stream around each solve, L2 flushed (256 MiB write) between steps
  outside the events.
* e2e: the same metric through the C ABI with host (pinned) buffers: the
  chunked pool pipeline (odegpu_pipeline_run, 8 chunks, copy-in / kernels /
  copy-out streams overlapped) — H2D of the pool, solve, D2H of time
  domains / state / accessories / outcome records into host arrays, per
  step, wall-clock.
* roofline: FP64-pipe lane instructions per trial step (SURVEY.md §8d
  algorithmic count) / solve-kernel time vs the DFMA microbenchmark peak.
* cpu_baseline: the reference solver (oracle/_ref, compiled from the
  reference's own sources) timed on this box's host cores on a bounded
  strided sample of the same workload.

Multi-GPU (torchrun): weak scaling; rank r owns rows [r*1024, (r+1)*1024) of a
(1024*N) x 1024 grid; no collective on the data path; the barrier and a MAX
all-reduce of the timed region are the only communication.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
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


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg2", choices=sorted(workloads.CONFIGS) + ["cfg5"])
    ap.add_argument("--log2n", type=int, default=24, help="cfg5: Keller-Miksis pool of 2^log2n systems")
    ap.add_argument("--strong", action="store_true",
                    help="cfg5 under torchrun: the 2^log2n pool is split over the ranks (default: each rank "
                         "integrates 2^log2n systems)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--e2e-chunks", type=int, default=0, help="pipeline chunks for e2e (0 = by pool size)")
    ap.add_argument("--cpu-sample", type=int, default=0, help="systems in the CPU sample (0 = auto)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def make_workload(name: str, rank: int, world: int, args=None):
    """Rank-local slice of the weak-scaling grid (cfg5 --strong: a contiguous
    slice of one fixed pool, odegpu_slice's split)."""
    if name == "cfg5":
        wl = workloads.cfg5(args.log2n)
        if world > 1 and args.strong:
            lo, hi = pkg.slice_range(wl.n, world, rank)
            wl = wl.subset(slice(lo, hi))
            wl.description += f"; rank {rank}/{world} slice [{lo}, {hi}) (strong scaling)"
        elif world > 1:
            wl.description += f"; rank {rank}/{world} replica (weak scaling)"
        return wl
    if name == "cfg2" and world > 1:
        full_k = workloads.param_range(0.2, 0.3, 1024 * world)
        wl = workloads.cfg2(1024, 1024)
        k = np.repeat(full_k[rank * 1024:(rank + 1) * 1024], 1024)
        wl.p[0] = k
        wl.description += f"; rank {rank}/{world} slice of a {1024 * world}x1024 grid"
        return wl
    wl = workloads.CONFIGS[name]()
    if world > 1:  # replicate other configs with a disjoint shift of the first parameter row
        wl.description += f"; rank {rank}/{world} replica"
    return wl


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


def cpu_baseline(wl, sample: int, iterations: int = 1):
    """Reference solver (oracle/_ref) on all host cores, bounded strided sample."""
    from oracle import pyoracle

    if not pyoracle.available("reference"):
        return None
    cores = pyoracle.host_cores()
    sub = wl.strided(sample)
    r = pyoracle.solve_workload("reference", sub, iterations, workers=cores)
    steps = int(r["outcomes"]["accepted_steps"].sum() + r["outcomes"]["rejected_steps"].sum())
    # outcomes hold the last iteration only; scale by iterations for the rate
    rate = steps * iterations / r["seconds"]
    return {"value": rate, "unit": UNIT, "cores": cores, "kind": "reference",
            "sample": f"{sub.n} of {wl.n} systems (evenly strided), {iterations} solve() iteration(s), "
                      f"{r['seconds']:.2f} s wall, ODENSEMBLE worker_count={cores}",
            "systems_per_s": sub.n * iterations / r["seconds"]}


def run_reference_arm(args, rank, world):
    """--impl reference: the reference CPU solver on this box's host cores."""
    if rank != 0:
        return
    from oracle import pyoracle

    wl = workloads.cfg5(args.log2n) if args.config == "cfg5" else workloads.CONFIGS[args.config]()
    if not pyoracle.available("reference"):
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libodref.so not built"}))
        return
    cores = pyoracle.host_cores()
    sample = args.cpu_sample or {"cfg1": 46080, "cfg2": 1 << 20, "cfg3": 1 << 17, "cfg4": 1 << 18,
                                 "cfg5": 1 << 17}[args.config]
    sub = wl.strided(sample)
    # like the GPU arm, every step solves the sample from its initial
    # conditions (iterating cfg2 in place hits the reference's secant Zeno
    # loop from the 3rd period on)
    for _ in range(args.warmup):
        td, y, p, acc = sub.arrays()
        pyoracle.solve("reference", sub.model, td, y, p, acc, algorithm=sub.algorithm, dt=sub.dt, iterations=1,
                       workers=cores)
    total_steps, total_s = 0, 0.0
    for _ in range(args.steps):
        td, y, p, acc = sub.arrays()
        oc, secs, _ = pyoracle.solve("reference", sub.model, td, y, p, acc, algorithm=sub.algorithm, dt=sub.dt,
                                     iterations=1, workers=cores)
        total_steps += int(oc["accepted_steps"].sum() + oc["rejected_steps"].sum())
        total_s += secs
    value = total_steps / total_s
    desc = f"{sub.n} of {wl.n} systems (evenly strided) per step, reference solve() on {cores} threads"
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total_s / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": wl.name, "description": wl.description, "sample": desc},
        "systems_per_s": sub.n * args.steps / total_s,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference", "sample": desc},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


_T0 = time.time()


def log(msg: str):
    print(f"[bench +{time.time() - _T0:7.1f}s] {msg}", file=sys.stderr, flush=True)


def main():
    args = parse()
    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist

        import torch

        # one rank per GPU: NCCL; ranks sharing a GPU (single-GPU test runs): gloo
        shared = torch.cuda.device_count() < world
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
    log(f"torch ready, rank {rank}/{world} on cuda:{local}")
    wl = make_workload(args.config, rank, world, args)
    n = wl.n
    td, y, p, acc = wl.arrays()
    pool = pkg.ProblemPool.from_arrays(td, y, p, acc)
    batch = pkg.SolverBatch(pkg.make_batch_dims(n, wl.model.dims()), device=device)
    stream = torch.cuda.Stream(device=device)
    batch.set_stream(stream.cuda_stream)
    cfg = pkg.SolverConfig(wl.algorithm, wl.dt)
    pkg.linear_set(batch, pool, pkg.LinearCopySpec(0, 0, n))
    # Every step integrates the synthetic batch from its initial conditions:
    # a pristine copy stays resident in HBM and is restored device-to-device
    # outside the timed events. (Iterating cfg2 in place is not an option:
    # from the 3rd forcing period on, 5 of its 2^20 systems enter a
    # secant/relocation Zeno loop — theta clamps to h*1e-12 forever — in the
    # reference solver itself.)
    pristine = pkg.SolverBatch(pkg.make_batch_dims(n, wl.model.dims()), device=device)
    pkg.batch_copy(pristine, batch)

    log(f"{wl.name}: {n} systems resident")
    peak_lane, _ = pkg.dfma_peak(device)
    log(f"DFMA peak {peak_lane:.4e} lane-DFMA/s")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{device}")

    for _ in range(args.warmup):
        pkg.batch_copy(batch, pristine)
        pkg.solve(batch, wl.model, cfg)

    # ---------------- timed region (device-resident batch)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    launches0 = batch.launch_count()
    ev_ms, kern_ms, steps_total, sys_total, max_trial = [], [], 0, 0, 0
    with ClockSampler(device) as clocks:
        for _ in range(args.steps):
            pkg.batch_copy(batch, pristine)  # initial conditions, outside the events
            with torch.cuda.stream(stream):
                flush.fill_(1)  # L2 flush between steps, outside the events
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            pkg.solve(batch, wl.model, cfg)
            e1.record(stream)
            e1.synchronize()
            ev_ms.append(e0.elapsed_time(e1))
            kern_ms.append(batch.last_kernel_ms())
            certified = batch.trig_certified()
            d = batch.diagnostics()
            steps_total += d["accepted_steps"] + d["rejected_steps"]
            max_trial = max(max_trial, d["max_trial_steps"])
            sys_total += n
    launches = batch.launch_count() - launches0 - args.steps  # minus the diagnostics tallies
    torch.cuda.synchronize()
    elapsed = sum(ev_ms) / 1e3
    kernel_s = sum(kern_ms) / 1e3
    if world > 1:
        import torch.distributed as dist

        t = torch.tensor([elapsed, kernel_s], dtype=torch.float64, device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed, kernel_s = float(t[0]), float(t[1])
        c = torch.tensor([steps_total, sys_total], dtype=torch.float64, device=red_dev)
        dist.all_reduce(c, op=dist.ReduceOp.SUM)
        steps_total, sys_total = int(c[0]), int(c[1])

    value = steps_total / elapsed
    achieved = steps_total * wl.instr_per_step / kernel_s  # lane FP64-pipe instr/s (all ranks)
    peak_total = peak_lane * world

    log(f"timed region done: {steps_total} trial steps in {elapsed:.4f} s")
    # the same solve in natural fetch order (outside the timed region), for
    # the fetch_order note in config: the timed steps take up systems
    # longest-first by the previous solve's trial steps (AUTO policy)
    cost_order = wl.algorithm == abi.RKCK45
    natural_ms = None
    if cost_order:
        batch.set_fetch_order(abi.FETCH_NATURAL)
        pkg.batch_copy(batch, pristine)
        pkg.solve(batch, wl.model, cfg)
        natural_ms = batch.last_kernel_ms()
        batch.set_fetch_order(abi.FETCH_AUTO)
    # ---------------- e2e: through the C ABI with host buffers, per step
    h_td = torch.empty(2 * n, dtype=torch.float64, pin_memory=True).numpy()
    h_y = torch.empty(y.size, dtype=torch.float64, pin_memory=True).numpy()
    h_p = torch.empty(p.size, dtype=torch.float64, pin_memory=True).numpy()
    h_a = torch.empty(max(acc.size, 1), dtype=torch.float64, pin_memory=True).numpy()[: acc.size]
    h_td[:], h_y[:], h_p[:], h_a[:] = td, y, p, acc
    pin_pool = pkg.ProblemPool.from_arrays(td, y, p, acc)
    pin_pool._td, pin_pool._state, pin_pool._params, pin_pool._acc = h_td, h_y, h_p, h_a
    o_y = torch.empty(y.size, dtype=torch.float64, pin_memory=True).numpy()
    o_td = torch.empty(2 * n, dtype=torch.float64, pin_memory=True).numpy()
    o_a = torch.empty(max(acc.size, 1), dtype=torch.float64, pin_memory=True).numpy()[: acc.size]
    lib = abi.load()
    h2d = (h_td.nbytes + h_y.nbytes + h_p.nbytes + h_a.nbytes)
    d2h = o_y.nbytes + o_td.nbytes + o_a.nbytes + n * abi.OUTCOME_DTYPE.itemsize
    e2e_steps, e2e_s = 0, 0.0
    outc = torch.zeros(n * abi.OUTCOME_DTYPE.itemsize, dtype=torch.uint8, pin_memory=True).numpy().view(
        abi.OUTCOME_DTYPE)
    if world > 1:
        torch.distributed.barrier()
    # the chunked pool pipeline: chunks through a 3-stage copy-in / kernels /
    # copy-out pipeline (odegpu_pipeline_run); device batches and pinned
    # staging are allocated once, like a scan driver would. Chunk count
    # (scripts/e2e_chunks.py): ~64 Ki systems per chunk, 2..8 chunks for the
    # transfer-bound cheap models, up to 16 for Keller-Miksis
    n_chunks = args.e2e_chunks or int(min(max(round(n / 65536), 2), 16 if wl.instr_per_step > 500 else 8))
    cap = max(1, -(-n // n_chunks))
    pipe = pkg.api.Pipeline(wl.model, cap, device)
    outs = (o_td, o_y, o_a, outc)
    pipe.run(pin_pool, cfg, 1, out_arrays=outs)  # warm-up (first-touch of the output pages)
    for _ in range(args.e2e_steps):
        t0 = time.perf_counter()
        pipe.run(pin_pool, cfg, 1, out_arrays=outs)
        e2e_s += time.perf_counter() - t0
        e2e_steps += int(outc["accepted_steps"].sum() + outc["rejected_steps"].sum())
    pipe.close()
    if world > 1:
        import torch.distributed as dist

        t = torch.tensor([e2e_s, e2e_steps], dtype=torch.float64, device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t[0])
        e2e_steps = e2e_steps * world  # weak scaling: every rank did its share
    e2e_value = e2e_steps / e2e_s

    if rank != 0:
        if world > 1:
            torch.distributed.barrier()
            torch.distributed.destroy_process_group()
        return

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        sample = args.cpu_sample or {"cfg1": 46080, "cfg2": 1 << 20, "cfg3": 1 << 18, "cfg4": 1 << 19,
                                     "cfg5": 1 << 18}[args.config]
        log(f"e2e done ({e2e_value:.4e} steps/s); CPU baseline on {sample} systems")
        cpu = cpu_baseline(wl, sample)

    traffic = load_traffic(wl.name)
    per_launch_s = kernel_s / args.steps
    hbm_bytes = n * 8 * (2 * 2 + 2 * wl.model.dims().system_dim + wl.model.dims().param_count
                         + 2 * wl.model.dims().accessory_count) + n * 49
    out = {
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": 1e3 * elapsed / args.steps,
        "higher_is_better": True,
        "scaling": "strong" if (args.config == "cfg5" and args.strong) else "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic",
        "config": {
            "workload": wl.name if args.config != "cfg5" else f"cfg5_keller_miksis_2^{args.log2n}",
            "description": wl.description,
            "systems_per_gpu": n,
            "step": "one solve() over the batch (one forcing period for cfg1/cfg2, one collapse / section-to-"
                    "section iteration for cfg3/cfg4)",
            "algorithm": "RK4" if wl.algorithm == abi.RK4 else "RKCK45",
            "l2": "flushed between steps (256 MiB write outside the timed events)",
            "parallelism": f"replicas{world}" if world > 1 else "single GPU",
            "trig_path": "certified (branch-free, include/odegpu/trig.hpp)" if certified else "general",
            "fetch_order": ("longest first by each system's trial steps in the batch's previous solve (AUTO "
                            "policy; here the previous timed step, i.e. the same solve: exact costs. Ordered by "
                            "the previous iteration of an in-place scan instead, the gain is 5-7% rather than "
                            "8-11% - DESIGN.md 3.1)") if cost_order else "natural (fixed step: equal costs)",
            "natural_order_kernel_ms": natural_ms,
        },
        "systems_per_s": sys_total / elapsed,
        "trial_steps_per_system_step": steps_total / max(sys_total, 1),
        "max_trial_steps_one_system": max_trial,
        "gpu_launches": launches,
        "kernel_ms_per_step": 1e3 * per_launch_s,
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
            "hbm_gbs": hbm_bytes / per_launch_s / 1e9,
        },
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "steps": args.e2e_steps,
                "path": f"odegpu_pipeline_run over the pinned host pool: {n_chunks} chunks, H2D / kernels / D2H of td, "
                        "state, accessories and outcome records on separate streams (4 chunks in flight), "
                        "into host arrays, wall-clock"},
        "cpu_baseline": cpu,
        "clocks": clocks.summary(),
    }
    print(json.dumps(out))
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
