#!/bin/bash
# A/B of the libraries in paper_1810_03931_b200/lib/variants/: solve-kernel
# time per config (scripts/quick_perf.py, natural fetch order unless FETCH
# is set), two interleaved rounds. -> gpurun_out/ab.jsonl
mkdir -p gpurun_out
rm -f gpurun_out/ab.jsonl
python -c "import torch; torch.zeros(1).cuda()" 2>/dev/null
for round in 1 2; do
  for v in paper_1810_03931_b200/lib/variants/*.so; do
    ODEGPU_LIB=$v FETCH=${FETCH:-0} timeout 300 python scripts/quick_perf.py ${CONFIGS:-cfg2 cfg4 cfg1} >> gpurun_out/ab.jsonl 2>> gpurun_out/ab.err
  done
done
python - <<'PY'
import json, collections
r = collections.defaultdict(list)
for ln in open("gpurun_out/ab.jsonl"):
    d = json.loads(ln); r[(d["name"], d["lib"])].append(d["best_ms"])
for (n, l), v in sorted(r.items()):
    print(f"{n} {l:28s} best {min(v):.4f} ms  all {v}")
PY
