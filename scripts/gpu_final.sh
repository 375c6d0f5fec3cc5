#!/bin/bash
# Evidence run: GPU suite, smoke, C++ host tests, bench lines (default = the
# driver's command, per-config, reference arm), ncu captures + launch list.
O=gpurun_out/${TAG:-final}
mkdir -p $O
python -c "import torch; torch.zeros(1).cuda()" 2>/dev/null
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $O/nvsmi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "rc=$?" >> $O/smoke.txt
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1; echo "rc=$?" >> $O/pytest_gpu.txt
./build/cpp/test_host_api > $O/cpp_tests.txt 2>&1; echo "cpp rc=$?" >> $O/cpp_tests.txt
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
for c in cfg1 cfg2 cfg3 cfg4; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
done
TAG=${TAG:-final} CONFIGS="cfg5 cfg2 cfg3 cfg4" bash scripts/gpu_ncu_r02.sh > $O/ncu.log 2>&1
tail -3 $O/pytest_gpu.txt; tail -1 $O/cpp_tests.txt; tail -2 $O/smoke.txt
for f in $O/bench_*.json; do python -c "
import json
d=json.load(open('$f')); r=d.get('roofline') or {}; e=d.get('e2e') or {}
print('$f', '%.4g'%d['value'], 'frac', r.get('frac'), 'e2e %.4g'%e.get('value',0), 'clocks', (d.get('clocks') or {}).get('sm_mhz'))" || tail -3 ${f%.json}.err; done
ls $O
