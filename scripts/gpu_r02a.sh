#!/bin/bash
# Round 2, first GPU pass: tests, the new default bench (cfg5 2^24 in place),
# builder-run lines for cfg1-4, the parity build's speed, and the full-size
# parity gate for both builds.
O=gpurun_out/r02a
mkdir -p $O
nvidia-smi > $O/nvidia_smi.txt 2>&1
lscpu > $O/lscpu.txt 2>&1
python -c "import torch; torch.zeros(1).cuda()" 2>/dev/null
timeout 300 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
for c in cfg2 cfg3 cfg4 cfg1; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
done
ODEGPU_BUILD=parity timeout 900 python bench.py --no-cpu-baseline --e2e-steps 1 > $O/bench_parity_build.json 2> $O/bench_parity_build.err
timeout 2400 python scripts/parity_fullsize.py --configs cfg2,cfg4,cfg3,cfg1,cfg5 --out $O/parity > $O/parity_fast.txt 2>&1
ODEGPU_BUILD=parity timeout 1200 python scripts/parity_fullsize.py --configs cfg2,cfg4,cfg3,cfg1,cfg5 --out $O/parity > $O/parity_parity.txt 2>&1
tail -3 $O/pytest_gpu.txt; cat $O/bench_default.json; tail -2 $O/bench_default.err
