#!/bin/bash
# GPU suite + smoke + bench lines after the streaming pipeline
O=gpurun_out/${TAG:-r02v}
mkdir -p $O
python -c "import torch; torch.zeros(1).cuda()" 2>/dev/null
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "rc=$?" >> $O/smoke.txt
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1; echo "rc=$?" >> $O/pytest_gpu.txt
tail -3 $O/pytest_gpu.txt
./build/cpp/test_host_api > $O/cpp_tests.txt 2>&1; echo "cpp rc=$?" >> $O/cpp_tests.txt; tail -1 $O/cpp_tests.txt
for c in cfg1 cfg2 cfg4; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
for f in $O/bench_*.json; do python -c "
import json
d=json.load(open('$f')); print('$f', round(d['value']/1e9,3), 'G/s kernel', round(d['kernel_ms_per_step'],3), 'ms frac', round(d['roofline']['frac'],4), 'e2e', round(d['e2e']['value']/1e9,3), d['e2e'].get('mode'), (d.get('cpu_baseline') or {}).get('value'))" || tail -3 ${f%.json}.err; done
