#!/bin/bash
# Tuning builds: libodegpu with a forced __launch_bounds__ min-blocks value,
# into paper_1810_03931_b200/lib/variants/libodegpu_mb<N>.so (load with ODEGPU_LIB=...).
set -e
cd "$(dirname "$0")/.."
NVFLAGS="-std=c++20 --expt-relaxed-constexpr -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -Xcompiler -fPIC -Iinclude -Ipaper_1810_03931_b200/csrc"
mkdir -p paper_1810_03931_b200/lib/variants
for mb in "$@"; do
  od=build/var_mb$mb; mkdir -p $od
  for f in paper_1810_03931_b200/csrc/*.cu; do
    b=$(basename $f .cu)
    nvcc $NVFLAGS -DODEGPU_MIN_BLOCKS=$mb -c -o $od/$b.o $f &
  done
  wait
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC -o paper_1810_03931_b200/lib/variants/libodegpu_mb$mb.so $od/*.o
done
