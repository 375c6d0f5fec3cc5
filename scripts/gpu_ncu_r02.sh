#!/bin/bash
# ncu --set full (clocks NOT locked: --clock-control none) of the solve kernel
# in the bench's own step shape: cfg2 from the initial conditions (natural
# order), cfg3 / cfg5 the 4th in-place iteration (previous-iteration order).
O=gpurun_out/${TAG:-r02c}
mkdir -p $O
python -c "import torch; torch.zeros(1).cuda()" 2>/dev/null
run() { # name skip args...
  local name=$1 skip=$2; shift 2
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:guarded_solve -s $skip -c 1 -f \
      -o $O/prof_$name python scripts/profile_one.py "$@" > $O/prof_$name.log 2>&1
}
for c in ${CONFIGS:-cfg2 cfg5 cfg3}; do
  case $c in
    cfg2) run cfg2 1 cfg2 ;;
    cfg5) run cfg5 4 cfg5 --inplace 3 ;;
    cfg3) run cfg3 4 cfg3 --inplace 3 ;;
    cfg4) run cfg4 4 cfg4 --inplace 3 ;;
    cfg1) run cfg1 4 cfg1 --inplace 3 ;;
  esac
done
# the bench's launch list with per-launch durations (clocks not locked)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-natural > $O/launches_bench.log 2>&1
ls -la $O
