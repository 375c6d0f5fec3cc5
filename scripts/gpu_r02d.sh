#!/bin/bash
O=gpurun_out/${TAG:-r02d}
mkdir -p $O
python -c "import torch; torch.zeros(1).cuda()" 2>/dev/null
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.txt 2>&1; echo "rc=$?" >> $O/pytest_gpu.txt
timeout 900 python bench.py --no-cpu-baseline > $O/bench_default.json 2> $O/bench_default.err
for c in ${CONFIGS:-cfg2 cfg3 cfg4 cfg1}; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
done
tail -3 $O/pytest_gpu.txt
for f in $O/bench_*.json; do python -c "
import json,sys
d=json.load(open('$f')); print('$f', round(d['value']/1e9,3), 'G/s kernel', round(d['kernel_ms_per_step'],3), 'ms frac', round(d['roofline']['frac'],4), 'e2e', round(d['e2e']['value']/1e9,3), d['config'].get('natural_order'))"; done
