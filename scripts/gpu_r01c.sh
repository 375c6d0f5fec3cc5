#!/bin/bash
# variants + tests + ncu of cfg3 and cfg2 with the current default build
bash scripts/gpu_variants.sh
CONFIGS="cfg3 cfg2" bash scripts/gpu_ncu.sh > gpurun_out/ncu.log 2>&1
ls gpurun_out/*.ncu-rep
