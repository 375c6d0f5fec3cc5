#!/bin/bash
# ncu --set full (clocks not locked) of one solve kernel with source
# correlation; exports the raw and SASS-source pages as CSV next to the report.
# usage: CONFIGS="cfg2 cfg1" TAG=r02f bash scripts/gpu_ncu_src.sh
O=gpurun_out/${TAG:-r02f}
mkdir -p $O
python -c "import torch; torch.zeros(1).cuda()" 2>/dev/null
for c in ${CONFIGS:-cfg2}; do
  case $c in
    cfg2) skip=1; args="cfg2" ;;
    cfg1) skip=4; args="cfg1 --inplace 3" ;;
    cfg4) skip=4; args="cfg4 --inplace 3" ;;
    cfg3) skip=4; args="cfg3 --inplace 3" ;;
  esac
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:guarded_solve -s $skip -c 1 -f \
      -o $O/prof_$c python scripts/profile_one.py $args > $O/prof_$c.log 2>&1
  ncu -i $O/prof_$c.ncu-rep --page raw --csv > $O/raw_$c.csv 2>/dev/null
  ncu -i $O/prof_$c.ncu-rep --page source --csv --print-source sass > $O/src_$c.csv 2>/dev/null
done
ls -la $O
