#!/bin/bash
# Perf of the tuning variants + the default build; then the GPU test suite.
mkdir -p gpurun_out
rm -f gpurun_out/variants.jsonl
for v in paper_1810_03931_b200/lib/variants/*.so paper_1810_03931_b200/lib/libodegpu.so; do
  ODEGPU_LIB=$v timeout 300 python scripts/quick_perf.py ${CONFIGS:-cfg2 cfg3 cfg4 cfg1} >> gpurun_out/variants.jsonl 2>> gpurun_out/variants.err
done
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.txt 2>&1
./build/cpp/test_host_api > gpurun_out/cpp_tests.txt 2>&1; echo "cpp rc=$?" >> gpurun_out/cpp_tests.txt
tail -3 gpurun_out/pytest_gpu.txt; tail -1 gpurun_out/cpp_tests.txt; cat gpurun_out/variants.jsonl
