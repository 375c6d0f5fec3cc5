#!/bin/bash
# One GPU session: C++ API tests, bench, ncu captures of the solve kernel.
set -u
mkdir -p gpurun_out
python -c "import torch; torch.zeros(1).cuda()" 2>/dev/null
./build/cpp/test_host_api > gpurun_out/cpp_tests.txt 2>&1; echo "cpp rc=$?" >> gpurun_out/cpp_tests.txt
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
for c in ${CONFIGS:-cfg3 cfg2 cfg4 cfg1}; do
  timeout 300 ncu --set full --import-source on -k regex:guarded_solve -s 1 -c 1 -f -o gpurun_out/prof_$c \
      python scripts/profile_one.py $c > gpurun_out/prof_$c.log 2>&1
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/launches_bench.log 2>&1
timeout 300 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.txt 2>&1
tail -2 gpurun_out/pytest_gpu.txt; tail -1 gpurun_out/cpp_tests.txt; cat gpurun_out/bench_cfg2.json | head -c 600
