#!/bin/bash
# Perf of the tuning variants + the default build (no tests).
mkdir -p gpurun_out
rm -f gpurun_out/variants.jsonl
for v in paper_1810_03931_b200/lib/variants/*.so paper_1810_03931_b200/lib/libodegpu.so; do
  ODEGPU_LIB=$v timeout 300 python scripts/quick_perf.py ${CONFIGS:-cfg2 cfg3 cfg4 cfg1} >> gpurun_out/variants.jsonl 2>> gpurun_out/variants.err
done
cat gpurun_out/variants.jsonl
