"""The glibc libm restatement (include/odegpu/device/glibm.h) evaluated ON
THE DEVICE equals the host's glibc bit for bit — the property the
exact-parity build (make parity) rests on. Inputs cover the regimes the
solver meets: Duffing forcing phases, Keller-Miksis excitation phases, the
controller's error ratios and the bubble's 1/y1 powers."""
import ctypes as C
from pathlib import Path

import numpy as np
import pytest

from test_gpu_dmath import run, same_bits

pytestmark = pytest.mark.gpu

HOST = Path(__file__).resolve().parents[1] / "oracle" / "_build" / "libglibm_host.so"


@pytest.fixture(scope="module")
def libm():
    L = C.CDLL(str(HOST))
    P = C.c_void_p
    L.libm_cos_batch.argtypes = [C.c_long, P, P]
    L.libm_sincos_batch.argtypes = [C.c_long, P, P, P]
    L.libm_pow_batch.argtypes = [C.c_long, P, P, P]
    return L


def phases(rng):
    return np.concatenate([
        rng.uniform(-1e-6, 1e-6, 20_000), rng.uniform(-0.9, 0.9, 100_000), rng.uniform(0.8, 2.5, 100_000),
        rng.uniform(-7000, 7000, 200_000), rng.uniform(-1e8, 1e8, 50_000),
        np.array([0.0, -0.0, 1e-300, 5e-324, np.pi / 2, np.pi, 2 * np.pi, np.inf, -np.inf, np.nan]),
    ])


def test_device_cos_equals_glibc(libm):
    x = phases(np.random.default_rng(3))
    mine, _ = run(10, x)
    host = np.empty_like(x)
    libm.libm_cos_batch(x.size, x.ctypes.data, host.ctypes.data)
    ok, bad = same_bits(mine, host)
    assert ok, f"{bad} device cos results differ from glibc"


def test_device_sincos_equals_glibc(libm):
    x = phases(np.random.default_rng(4))
    mine, _ = run(11, x)
    s, c = np.empty_like(x), np.empty_like(x)
    libm.libm_sincos_batch(x.size, x.ctypes.data, s.ctypes.data, c.ctypes.data)
    ok, bad = same_bits(mine, np.concatenate([s, c]))
    assert ok, f"{bad} device sincos results differ from glibc"


def test_device_pow_equals_glibc(libm):
    rng = np.random.default_rng(5)
    x = np.concatenate([np.exp(rng.uniform(np.log(1e-12), np.log(1e12), 200_000)),
                        np.exp(rng.uniform(np.log(1e-3), np.log(1e4), 200_000)),
                        np.exp(rng.uniform(-700, 700, 50_000)),
                        np.array([0.0, 1.0, np.inf, np.nan, 5e-324, 2.2e-308])])
    y = np.concatenate([np.full(200_000, -0.2), np.full(200_000, 4.2), rng.uniform(-4, 4, 50_000),
                        np.full(6, -0.2)])
    mine, _ = run(12, x, y)
    host = np.empty_like(x)
    with np.errstate(all="ignore"):
        libm.libm_pow_batch(x.size, x.ctypes.data, y.ctypes.data, host.ctypes.data)
    ok, bad = same_bits(mine, host)
    assert ok, f"{bad} device pow results differ from glibc"
