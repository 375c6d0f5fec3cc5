"""The trig certificate (include/odegpu/trig.hpp): a batch runs the
branch-free trig instantiation only when every system's trig arguments are
provably below 2^31, and both instantiations match the oracle."""
import numpy as np
import pytest

import paper_1810_03931_b200 as pkg
import parity
from oracle import pyoracle
from paper_1810_03931_b200 import workloads

pytestmark = pytest.mark.gpu


def run(wl):
    td, y, p, acc = wl.arrays()
    pool = pkg.ProblemPool.from_arrays(td, y, p, acc)
    b = pkg.SolverBatch(pkg.make_batch_dims(wl.n, wl.model.dims()))
    pkg.linear_set(b, pool, pkg.LinearCopySpec(0, 0, wl.n))
    pkg.solve(b, wl.model, pkg.SolverConfig(wl.algorithm, wl.dt))
    out = dict(y=b.state(), acc=b.accessories(), outcomes=b.outcomes(), certified=b.trig_certified())
    b.close()
    return out


def check(wl, got):
    ref = pyoracle.solve_workload("port", wl, iterations=1)
    for k in parity.COUNT_FIELDS:
        assert np.array_equal(got["outcomes"][k], ref["outcomes"][k]), k
    err = parity.rel_err(got["y"], ref["y"], 1e-9)
    assert err.max() <= 1e-9, err.max()


@pytest.mark.parametrize("cfg", ["cfg1", "cfg2"])
def test_in_range_batch_is_certified(cfg):
    wl = workloads.CONFIGS[cfg]().strided(2048)
    got = run(wl)
    assert got["certified"], "omega*t <= 2 pi must certify"
    check(wl, got)


def test_one_large_argument_uncertifies_the_batch():
    """omega = 1e9 on a [0, 4] domain puts omega*t beyond 2^31 for one
    system: the whole batch takes the general path (libdevice Payne-Hanek
    beyond 2^31), and still matches the oracle (glibc cos)."""
    wl = workloads.cfg1().strided(1024)
    wl.td[1, :] = 4.0
    wl.p[3, 17] = 1e9
    got = run(wl)
    assert not got["certified"]
    check(wl, got)
    wl.p[3, 17] = 1.0
    assert run(wl)["certified"]


def test_keller_miksis_certificate():
    wl = workloads.cfg3().strided(512)
    got = run(wl)
    assert got["certified"]  # 2 pi * 1e6 < 2^31
    ref = pyoracle.solve_workload("port", wl, iterations=1)
    for k in parity.COUNT_FIELDS:
        assert np.array_equal(got["outcomes"][k], ref["outcomes"][k]), k


def test_models_without_trig_report_uncertified():
    wl = workloads.cfg4().strided(256)
    assert not run(wl)["certified"]
