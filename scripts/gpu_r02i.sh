#!/bin/bash
O=gpurun_out/${TAG:-r02i}
mkdir -p $O
python -c "import torch; torch.zeros(1).cuda()" 2>/dev/null
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1; echo "rc=$?" >> $O/pytest_gpu.txt

for c in cfg3 cfg4 cfg5_22; do timeout 300 python scripts/pool_cluster_perf.py $c 4; timeout 300 python scripts/pool_cluster_perf.py $c 8 >> $O/pool_cluster.jsonl 2>> $O/pool_cluster.err; done
tail -3 $O/pytest_gpu.txt; cat $O/e2e.txt; cat $O/pool_cluster.jsonl
