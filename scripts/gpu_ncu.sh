#!/bin/bash
# ncu --set full of the solve kernel for each config (second solve, full size).
mkdir -p gpurun_out
for c in ${CONFIGS:-cfg3 cfg2 cfg4 cfg1}; do
  timeout 400 ncu --set full --import-source on --clock-control none -k regex:guarded_solve -s 1 -c 1 -f -o gpurun_out/prof_$c \
      python scripts/profile_one.py $c > gpurun_out/prof_$c.log 2>&1
done
ls -la gpurun_out/*.ncu-rep
