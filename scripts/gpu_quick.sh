#!/bin/bash
mkdir -p gpurun_out
python -c "import torch; torch.zeros(1).cuda()" 2>/dev/null
timeout 300 python scripts/quick_perf.py cfg2 cfg3 cfg4 cfg1 > gpurun_out/perf_now.jsonl 2> gpurun_out/perf_now.err
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.txt 2>&1
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
tail -3 gpurun_out/pytest_gpu.txt; cat gpurun_out/perf_now.jsonl; python -c "
import json; d=json.load(open('gpurun_out/bench_quick.json')); print('bench', d['value'], d['roofline']['frac'], 'e2e', d['e2e']['value'])"
