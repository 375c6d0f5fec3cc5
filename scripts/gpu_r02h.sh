#!/bin/bash
# GPU tests + cfg2 / cfg5 bench lines after the detection log and the time-domain skip
O=gpurun_out/${TAG:-r02h}
mkdir -p $O
python -c "import torch; torch.zeros(1).cuda()" 2>/dev/null
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1; echo "rc=$?" >> $O/pytest_gpu.txt
./build/cpp/test_host_api > $O/cpp_tests.txt 2>&1; echo "cpp rc=$?" >> $O/cpp_tests.txt
timeout 600 python bench.py --config cfg2 --no-cpu-baseline > $O/bench_cfg2.json 2> $O/bench_cfg2.err
ODEGPU_PIPELINE_TRACE=1 timeout 900 python bench.py --no-cpu-baseline --steps 3 --e2e-steps 1 --no-natural > $O/bench_cfg5.json 2> $O/bench_cfg5.err
tail -3 $O/pytest_gpu.txt; tail -1 $O/cpp_tests.txt
for f in $O/bench_*.json; do python -c "
import json
d=json.load(open('$f')); print('$f', round(d['value']/1e9,3), 'G/s kernel', round(d['kernel_ms_per_step'],3), 'ms frac', round(d['roofline']['frac'],4), 'e2e', round(d['e2e']['value']/1e9,3), d['e2e']['d2h_bytes_per_step'])"; done
