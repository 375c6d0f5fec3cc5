#!/bin/bash
# Round 2: the glibc-restated parity build on the GPU — device libm vs host
# glibc, then the full-size parity gate for the parity build.
O=gpurun_out/r02b
mkdir -p $O
python -c "import torch; torch.zeros(1).cuda()" 2>/dev/null
timeout 300 python -m pytest tests/test_gpu_glibm.py tests/test_gpu_dmath.py -x -q > $O/pytest_glibm.txt 2>&1; echo "rc=$?" >> $O/pytest_glibm.txt
ODEGPU_BUILD=parity timeout 2400 python scripts/parity_fullsize.py --configs cfg2,cfg4,cfg3,cfg1,cfg5 --out $O/parity > $O/parity_parity.txt 2>&1
ODEGPU_BUILD=parity timeout 600 python bench.py --no-cpu-baseline --e2e-steps 1 > $O/bench_parity_build.json 2> $O/bench_parity_build.err
tail -3 $O/pytest_glibm.txt; cut -c1-400 $O/parity_parity.txt
