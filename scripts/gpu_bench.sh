#!/bin/bash
# Round deliverables: smoke, bench (ours + reference arm), ncu launch list of the bench command.
mkdir -p gpurun_out
python -c "import torch; torch.zeros(1).cuda()" 2>/dev/null
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.txt
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/clocks.csv &
SMI=$!
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
for c in cfg3 cfg4 cfg1; do timeout 600 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
kill $SMI
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/launches_bench.log 2>&1
tail -2 gpurun_out/smoke.txt; cat gpurun_out/bench_default.json; cat gpurun_out/bench_reference.json
