#!/bin/bash
# compute-sanitizer (memcheck, racecheck, initcheck) over the smoke solve and
# the parity / pipeline / scan tests at small sizes.
mkdir -p gpurun_out
rm -f gpurun_out/sanitize_summary.txt gpurun_out/san_*.txt
S=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck initcheck; do
  timeout 900 $S --tool $tool --error-exitcode 99 --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san_${tool}_smoke.txt 2>&1
  echo "$tool smoke rc=$?" >> gpurun_out/sanitize_summary.txt
done
timeout 1500 $S --tool memcheck --error-exitcode 99 --print-limit 20 python -m pytest -q -x tests/test_gpu_parity.py -k "golden" > gpurun_out/san_memcheck_parity.txt 2>&1
echo "memcheck parity golden rc=$?" >> gpurun_out/sanitize_summary.txt
timeout 900 $S --tool memcheck --error-exitcode 99 --print-limit 20 python -m pytest -q -x tests/test_gpu_pipeline.py tests/test_gpu_trig_certificate.py > gpurun_out/san_memcheck_pipeline.txt 2>&1
echo "memcheck pipeline+cert rc=$?" >> gpurun_out/sanitize_summary.txt
for tool in memcheck initcheck; do
  timeout 900 $S --tool $tool --error-exitcode 99 --print-limit 20 python -m pytest -q -x tests/test_gpu_fetch_order.py > gpurun_out/san_${tool}_fetch_order.txt 2>&1
  echo "$tool fetch order rc=$?" >> gpurun_out/sanitize_summary.txt
done
cat gpurun_out/sanitize_summary.txt; grep -h "ERROR SUMMARY" gpurun_out/san_*.txt
