#!/bin/bash
# Session re-entry check: perf of HEAD, GPU tests, bench line, ncu of cfg2/cfg3.
mkdir -p gpurun_out
python -c "import torch; torch.zeros(1).cuda()" 2>/dev/null
timeout 300 python scripts/quick_perf.py cfg2 cfg3 cfg4 cfg1 > gpurun_out/perf_now.jsonl 2> gpurun_out/perf_now.err
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.txt 2>&1
timeout 300 python bench.py > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
CONFIGS="cfg2 cfg3" bash scripts/gpu_ncu.sh > gpurun_out/ncu.log 2>&1
tail -3 gpurun_out/pytest_gpu.txt; cat gpurun_out/perf_now.jsonl; cat gpurun_out/bench_quick.json
