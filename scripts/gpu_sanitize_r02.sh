#!/bin/bash
# compute-sanitizer over this round's device paths at small sizes: the
# streaming pipeline, fused iterations, the detection log, the device pool.
O=gpurun_out/sanitizer_r02
mkdir -p $O
rm -f $O/summary.txt
S=/usr/local/cuda/bin/compute-sanitizer
run() { # tool name pytest-args...
  local tool=$1 name=$2; shift 2
  timeout 900 $S --tool $tool --error-exitcode 99 --print-limit 20 python -m pytest -q -x "$@" > $O/${tool}_${name}.txt 2>&1
  echo "$tool $name rc=$?" >> $O/summary.txt
}
run memcheck streaming tests/test_gpu_streaming.py
run racecheck streaming tests/test_gpu_streaming.py -k "equals_resident and cfg2"
run memcheck fused tests/test_gpu_fused.py
run memcheck detection_log tests/test_gpu_detection_log.py
run memcheck device_pool tests/test_gpu_device_pool.py
run initcheck device_pool tests/test_gpu_device_pool.py
cat $O/summary.txt; grep -h "ERROR SUMMARY" $O/*.txt
