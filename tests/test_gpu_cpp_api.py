"""Runs the C++ host-API test program (tests/cpp/test_host_api.cpp): the
reference test-suite's batch / driver / scan cases written against
include/odegpu/*.hpp, executed on the GPU through libodegpu."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
BIN = ROOT / "build" / "cpp" / "test_host_api"


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["test_host_api", "test_custom_model"])
def test_cpp_suite(name):
    """test_host_api: the reference's batch/driver/scan cases on the C++ API;
    test_custom_model: user-defined SystemModels compiled by nvcc through
    include/odegpu/device/custom.cuh (a clone of a built-in model must match
    it bitwise)."""
    binary = ROOT / "build" / "cpp" / name
    if not binary.exists():
        subprocess.run(["make", "-C", str(ROOT), "cpptests"], check=True)
    r = subprocess.run([str(binary)], capture_output=True, text=True, timeout=600)
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert ", 0 failed" in r.stdout


def test_cpp_host_api_compiles_with_plain_gxx(tmp_path):
    """The host API needs no CUDA toolchain on the caller side."""
    src = tmp_path / "t.cpp"
    src.write_text('#include "odegpu/odegpu.hpp"\nint main() { odegpu::models::ValveSystem v; '
                   'return static_cast<int>(v.dims().system_dim) - 3; }\n')
    subprocess.run(["g++", "-std=c++20", "-fsyntax-only", f"-I{ROOT / 'include'}", str(src)], check=True)
