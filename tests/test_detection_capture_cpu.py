"""The reference's own detection observer as a checker (oracle/_ref,
odref_capture_detections): what the device detection log is compared with
in tests/test_gpu_detection_log.py. CPU only."""
import numpy as np
import pytest

from oracle import pyoracle
from paper_1810_03931_b200 import workloads

pytestmark = pytest.mark.skipif(not pyoracle.available("reference"), reason="oracle/_ref not built")


@pytest.mark.parametrize("cfg,n", [("cfg2", 256), ("cfg4", 256)])
def test_reference_observer_records_every_detection(cfg, n):
    wl = workloads.CONFIGS[cfg]().strided(n)
    rec, pre, post, res = pyoracle.reference_detections(wl, 1)
    # one record per counted detection, grouped per system in call order
    per_sys = np.bincount(rec["system"], minlength=wl.n)
    assert np.array_equal(per_sys, res["outcomes"]["event_detections"])
    assert np.all(np.diff(rec["system"]) >= 0)
    for s in np.unique(rec["system"]):
        seq = rec["sequence"][rec["system"] == s]
        assert np.array_equal(seq, np.arange(seq.size))
    assert set(np.unique(rec["kind"])) <= {0, 1, 2}
    if cfg == "cfg4":  # ValveSystem's impact action (valve.hpp:66-76): y1 = 0, y2 = -r y2
        imp = rec["event_index"] == 1
        assert imp.any()
        assert np.all(post[imp, 0] == 0.0)
        p = wl.arrays()[2]
        r = p[rec["system"][imp] + 4 * wl.n]  # p = [kappa, delta, beta, q, r]
        assert np.array_equal(post[imp, 1], -r * pre[imp, 1])
    else:  # no action: the state is not touched
        assert np.array_equal(pre, post)
