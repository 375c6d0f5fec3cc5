#!/bin/bash
O=gpurun_out/r02w
mkdir -p $O
python -c "import torch; torch.zeros(1).cuda()" 2>/dev/null
timeout 300 python -m pytest tests/test_gpu_streaming.py -x -q 2>&1 | tail -2
CONFIGS="cfg2" TAG=r02w bash scripts/gpu_ncu_src.sh > /dev/null 2>&1
ls -la $O
