"""The exact-parity build (make parity: -fmad=false and glibc's libm restated
on the device, include/odegpu/device/glibm.h) reproduces the unmodified
reference solver BIT FOR BIT: time domains, states, accessories and every
outcome field of every system after every iteration, on strided samples of
all four configs and on the full-grid systems where the fast build's
rounding flips a knife-edge accept / reject decision (the full-size runs:
profiles/r02b/parity_fullsize_parity_build.jsonl), and on seeded random
off-grid inputs of every built-in model over two iterations."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
PARITY_LIB = ROOT / "paper_1810_03931_b200" / "lib" / "libodegpu_parity.so"

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cases():
    assert PARITY_LIB.exists(), "libodegpu_parity.so missing: make parity (built by __graft_entry__.build())"
    env = dict(os.environ, ODEGPU_BUILD="parity")
    env.pop("ODEGPU_LIB", None)
    r = subprocess.run([sys.executable, str(ROOT / "tests" / "parity_build_check.py")], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    return {d["case"]: d for d in (json.loads(l) for l in r.stdout.splitlines() if l.startswith("{"))}


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg4", "cfg3_knife_edges", "cfg5_knife_edges",
                                  "random_duffing_event", "random_duffing_accessory", "random_duffing_rk4",
                                  "random_valve", "random_bubble"])
def test_parity_build_bitwise_reference(cases, name):
    c = cases[name]
    assert c["td"] == 0 and c["y"] == 0 and c["acc"] == 0, c
    assert c["outcome_fields"] == 0, c
    assert all(m == 0 for m in c["per_iteration_count_mismatches"]), c


def test_knife_edge_system_takes_the_references_rejections(cases):
    # cfg3 system 541514 (1024 x 1024 grid, iteration 0): the reference takes
    # 4 rejected steps; the fast build's contracted arithmetic took 3
    assert cases["cfg3_knife_edges"]["rejected_steps"][0] == 4
