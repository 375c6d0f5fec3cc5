#!/bin/bash
# Quick GPU session: dmath bit-check, perf of the current build, full GPU tests.
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_dmath.py -q > gpurun_out/dmath.txt 2>&1
timeout 300 python scripts/quick_perf.py cfg2 cfg3 cfg4 cfg1 > gpurun_out/perf_now.jsonl 2> gpurun_out/perf_now.err
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.txt 2>&1
./build/cpp/test_host_api > gpurun_out/cpp_tests.txt 2>&1; echo "cpp rc=$?" >> gpurun_out/cpp_tests.txt
tail -3 gpurun_out/dmath.txt; tail -3 gpurun_out/pytest_gpu.txt; tail -1 gpurun_out/cpp_tests.txt; cat gpurun_out/perf_now.jsonl
