#!/bin/bash
# dmath checks, perf of the current build, GPU tests.
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_dmath.py -q > gpurun_out/dmath.txt 2>&1
timeout 300 python scripts/quick_perf.py cfg2 cfg3 cfg4 cfg1 > gpurun_out/perf_now.jsonl 2> gpurun_out/perf_now.err
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.txt 2>&1
tail -5 gpurun_out/dmath.txt; tail -3 gpurun_out/pytest_gpu.txt; cat gpurun_out/perf_now.jsonl
