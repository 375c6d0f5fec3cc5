"""The glibc libm restatement of the exact-parity build
(include/odegpu/device/glibm.h) against the live glibc libm the reference
links, bit for bit, on the host (oracle/_build/libglibm_host.so: the same
header compiled with -ffp-contract=off next to calls of libm's cos / sincos /
pow). The GPU side of the same comparison is tests/test_gpu_glibm.py."""
import ctypes as C
from pathlib import Path

import numpy as np
import pytest

LIB = Path(__file__).resolve().parents[1] / "oracle" / "_build" / "libglibm_host.so"


@pytest.fixture(scope="module")
def lib():
    if not LIB.exists():
        pytest.skip("oracle/_build/libglibm_host.so not built (make -C oracle oracle)")
    L = C.CDLL(str(LIB))
    P = C.c_void_p
    for f in ("glm_cos_batch", "libm_cos_batch"):
        getattr(L, f).argtypes = [C.c_long, P, P]
    for f in ("glm_sincos_batch", "libm_sincos_batch"):
        getattr(L, f).argtypes = [C.c_long, P, P, P]
    for f in ("glm_pow_batch", "libm_pow_batch"):
        getattr(L, f).argtypes = [C.c_long, P, P, P]
    return L


def same(a, b):
    return (a.view(np.uint64) == b.view(np.uint64)) | (np.isnan(a) & np.isnan(b))


# the reduction regimes of s_sin.c: |x| < 2^-27, < 0.855469 (do_cos / do_sin
# around a table point), < 2.426265 (pi/2 - |x|), < 105414350 (reduce_sincos)
TRIG_RANGES = [(0.0, 1e-8), (1e-8, 0.86), (0.85, 2.43), (2.4, 200.0), (200.0, 1e5), (1e5, 1.05e8)]


@pytest.mark.parametrize("lo,hi", TRIG_RANGES)
def test_cos_and_sincos_bitwise_glibc(lib, lo, hi):
    rng = np.random.default_rng(int(hi))
    x = rng.uniform(lo, hi, 200_000)
    x = np.concatenate([x, -x, [lo, hi, 0.855469, 2.426265, np.pi / 2, np.pi, 2 * np.pi]])
    a, b = np.empty_like(x), np.empty_like(x)
    lib.glm_cos_batch(x.size, x.ctypes.data, a.ctypes.data)
    lib.libm_cos_batch(x.size, x.ctypes.data, b.ctypes.data)
    assert np.all(same(a, b)), f"cos differs at {x[~same(a, b)][:5]}"
    s1, c1, s2, c2 = (np.empty_like(x) for _ in range(4))
    lib.glm_sincos_batch(x.size, x.ctypes.data, s1.ctypes.data, c1.ctypes.data)
    lib.libm_sincos_batch(x.size, x.ctypes.data, s2.ctypes.data, c2.ctypes.data)
    assert np.all(same(s1, s2)) and np.all(same(c1, c2))


def test_trig_special_values(lib):
    x = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 5e-324, 1e-300])
    a, b = np.empty_like(x), np.empty_like(x)
    lib.glm_cos_batch(x.size, x.ctypes.data, a.ctypes.data)
    lib.libm_cos_batch(x.size, x.ctypes.data, b.ctypes.data)
    assert np.all(same(a, b))


@pytest.mark.parametrize("case", ["controller", "keller_miksis", "wide", "random_bits", "integer_y"])
def test_pow_bitwise_glibc(lib, case):
    rng = np.random.default_rng(hash(case) % 2**32)
    n = 300_000
    if case == "controller":  # std::pow(ratio, -0.2), steppers.hpp:185
        x = np.exp(rng.uniform(np.log(1e-12), np.log(1e12), n))
        x[:4] = [0.0, 1.0, np.inf, np.nan]
        y = np.full(n, -0.2)
    elif case == "keller_miksis":  # pow(1/y1, 3 kappa), keller_miksis.hpp:90
        x = np.exp(rng.uniform(np.log(1e-3), np.log(1e4), n))
        y = np.full(n, 4.2)
    elif case == "wide":
        x = np.exp(rng.uniform(-700, 700, n))
        y = rng.uniform(-4, 4, n)
    elif case == "random_bits":
        x = rng.integers(0, 2**64, n, dtype=np.uint64).view(np.float64)
        y = rng.integers(0, 2**64, n, dtype=np.uint64).view(np.float64)
    else:
        x = rng.integers(0, 2**64, n, dtype=np.uint64).view(np.float64)
        y = np.round(rng.uniform(-10, 10, n))
    a, b = np.empty_like(x), np.empty_like(x)
    with np.errstate(all="ignore"):
        lib.glm_pow_batch(n, x.ctypes.data, y.ctypes.data, a.ctypes.data)
        lib.libm_pow_batch(n, x.ctypes.data, y.ctypes.data, b.ctypes.data)
    bad = ~same(a, b)
    assert not bad.any(), f"pow differs at x={x[bad][:3]}, y={y[bad][:3]}"
