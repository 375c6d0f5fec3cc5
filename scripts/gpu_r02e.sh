#!/bin/bash
# round-2 re-entry check: GPU tests + default bench + per-config bench + smoke
O=gpurun_out/${TAG:-r02e}
mkdir -p $O
python -c "import torch; torch.zeros(1).cuda()" 2>/dev/null
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/nvsmi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "rc=$?" >> $O/smoke.txt
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.txt 2>&1; echo "rc=$?" >> $O/pytest_gpu.txt
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
for c in ${CONFIGS:-cfg2 cfg3 cfg4 cfg1}; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
tail -3 $O/pytest_gpu.txt
for f in $O/bench_*.json; do python -c "
import json,sys
d=json.load(open('$f')); print('$f', d.get('value'), d.get('kernel_ms_per_step'), (d.get('roofline') or {}).get('frac'), (d.get('e2e') or {}).get('value'), d['config'].get('natural_order'))"; done
