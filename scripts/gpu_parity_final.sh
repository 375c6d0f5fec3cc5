#!/bin/bash
# Full-size parity gate on the final build: every system of cfg1-cfg5 at
# BASELINE size, both builds against the unmodified reference.
O=gpurun_out/r02ah
mkdir -p $O
python -c "import torch; torch.zeros(1).cuda()" 2>/dev/null
ODEGPU_BUILD=parity timeout 3000 python scripts/parity_fullsize.py --configs cfg1,cfg2,cfg4,cfg3,cfg5 --out $O/parity > $O/parity_build.txt 2>&1
timeout 1500 python scripts/parity_fullsize.py --configs cfg1,cfg2,cfg4,cfg3,cfg5 --out $O/fast > $O/fast_build.txt 2>&1
ls $O $O/parity $O/fast
