"""Summarise ncu captures (gpurun_out/prof_<cfg>.ncu-rep) into profiles/.

Writes profiles/ncu_summary.json (read by bench.py for roofline.traffic) and
profiles/<tag>_ncu_summary.md with the counters DESIGN.md argues from: FP64
pipe activity, issue activity, warps, registers, stall reasons, DRAM bytes,
local-memory traffic, lane efficiency and the dynamic instruction mix.

    python scripts/ncu_summary.py <tag> [cfg ...]      (reads gpurun_out/<tag>/prof_<cfg>.ncu-rep,
                                                         else gpurun_out/prof_<cfg>.ncu-rep)
"""
import csv
import io
import json
import re
import subprocess
import sys
from collections import Counter
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
NAMES = {"cfg1": "cfg1_duffing_rk4", "cfg2": "cfg2_duffing_rkck45_event", "cfg3": "cfg3_keller_miksis",
         "cfg4": "cfg4_valve", "cfg5": "cfg5_keller_miksis_2^24"}
METRICS = {
    "duration_ms": ("gpu__time_duration.sum", 1e-6),
    "fp64_pipe_active_pct": ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 1),
    "issue_active_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", 1),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    "registers": ("launch__registers_per_thread", 1),
    "grid": ("launch__grid_size", 1),
    "dram_read_bytes": ("dram__bytes_read.sum", 1),
    "dram_write_bytes": ("dram__bytes_write.sum", 1),
    "local_load_inst": ("smsp__sass_inst_executed_op_local_ld.sum", 1),
    "local_store_inst": ("smsp__sass_inst_executed_op_local_st.sum", 1),
    "lane_efficiency": ("smsp__thread_inst_executed_per_inst_executed.ratio", 1 / 32),
    "warp_instructions": ("smsp__inst_executed.sum", 1),
}
STALLS = ["wait", "no_instruction", "not_selected", "branch_resolving", "short_scoreboard", "math_pipe_throttle",
          "long_scoreboard", "mio_throttle", "dispatch_stall", "lg_throttle"]


def ncu(args):
    return subprocess.run(["ncu", "-i", *args], capture_output=True, text=True).stdout


def unit_scale(unit: str, value: float) -> float:
    """Normalise ncu's auto-scaled units (byte/Kbyte/Mbyte, nsecond/usecond...)."""
    u = unit.lower()
    table = {"kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9, "byte": 1.0, "us": 1e3, "usecond": 1e3, "ms": 1e6,
             "msecond": 1e6, "ns": 1.0, "nsecond": 1.0, "s": 1e9, "second": 1e9}
    return value * table.get(u, 1.0)


def raw_metrics(rep):
    rows = list(csv.reader(io.StringIO(ncu([str(rep), "--page", "raw", "--csv"]))))
    hdr, units, vals = rows[0], rows[1], rows[2]
    out = {}
    for h, u, v in zip(hdr, units, vals):
        try:
            out[h] = unit_scale(u, float(v.replace(",", "")))
        except ValueError:
            pass
    return out


def instruction_mix(rep):
    rows = list(csv.reader(io.StringIO(ncu([str(rep), "--page", "source", "--csv", "--print-source", "sass"]))))
    hdr = rows[1]
    i_src, i_exe = hdr.index("Source"), hdr.index("Instructions Executed")
    by = Counter()
    for r in rows[2:]:
        if len(r) <= i_exe:
            continue
        m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[i_src])
        if m and r[i_exe]:
            by[m.group(2)] += int(r[i_exe])
    total = sum(by.values())
    fp64 = sum(by[o] for o in ("DFMA", "DMUL", "DADD", "DSETP", "DMNMX"))
    return {"fp64_share_of_instructions": fp64 / max(total, 1),
            "top": {k: round(v / total, 4) for k, v in by.most_common(12)}}


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    cfgs = sys.argv[2:] or ["cfg1", "cfg2", "cfg3", "cfg4"]
    summary_path = ROOT / "profiles" / "ncu_summary.json"
    summary = json.loads(summary_path.read_text()) if summary_path.exists() else {}
    summary.setdefault("traffic_bytes_per_launch", {})
    summary.setdefault("kernels", {})
    lines = [f"# ncu summary ({tag})", "",
             "One `ncu --set full --clock-control none` capture of the solve kernel per workload (full "
             "BASELINE size, in the bench's step shape: cfg2 from the initial conditions, the others the 4th "
             "in-place iteration; scripts/gpu_ncu_r02.sh). Durations are of a kernel timed alone under replay.", ""]
    for c in cfgs:
        rep = ROOT / "gpurun_out" / tag / f"prof_{c}.ncu-rep"
        if not rep.exists():
            rep = ROOT / "gpurun_out" / f"prof_{c}.ncu-rep"
        if not rep.exists():
            continue
        m = raw_metrics(rep)
        d = {k: m.get(name, float("nan")) * f for k, (name, f) in METRICS.items()}
        d["stalls_per_issue"] = {s: round(m.get(f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio",
                                                float("nan")), 3) for s in STALLS}
        d.update(instruction_mix(rep))
        summary["kernels"][NAMES[c]] = {"tag": tag, **d}
        summary["traffic_bytes_per_launch"][NAMES[c]] = d["dram_read_bytes"] + d["dram_write_bytes"]
        lines.append(f"## {NAMES[c]}")
        for k, v in d.items():
            lines.append(f"* {k}: {v}")
        lines.append("")
    summary_path.write_text(json.dumps(summary, indent=1))
    (ROOT / "profiles" / f"{tag}_ncu_summary.md").write_text("\n".join(lines))
    print("\n".join(lines))


if __name__ == "__main__":
    main()
