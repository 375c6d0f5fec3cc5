"""bench.py's multi-GPU path (what the driver's scaling run launches) with two
ranks sharing this box's GPU: one process per rank under torchrun, the
rotated block split, NCCL-free (gloo) timing reductions on a shared device,
and the wall-clock region a shared GPU needs."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
pytestmark = pytest.mark.gpu


@pytest.mark.timeout(600)
def test_two_ranks_on_one_gpu_report_one_gpus_rate():
    cmd = [sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--allow-shared-gpu", "--config", "cfg4",
           "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--e2e-steps", "1"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=550, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1]
    d = json.loads(line)
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert d["config"]["systems"] == 524288 and d["config"]["systems_per_gpu"] < 524288
    assert "rotated" in d["config"]["parallelism"] and "wall clock" in d["config"]["timing"]
    assert d["gpu_launches"] >= 1 and d["value"] > 0 and d["e2e"]["value"] > 0
    # two time-sliced ranks cannot beat one GPU: the region is the wall clock
    # between barriers (per-rank CUDA-event spans would add their shares up)
    one = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--config", "cfg4", "--steps", "3", "--warmup",
                          "3", "--no-cpu-baseline", "--e2e-steps", "1", "--no-natural"],
                         capture_output=True, text=True, timeout=550, cwd=ROOT)
    assert one.returncode == 0, one.stderr[-3000:]
    single = json.loads([ln for ln in one.stdout.splitlines() if ln.startswith("{")][-1])
    assert d["value"] <= 1.15 * single["value"], (d["value"], single["value"])
