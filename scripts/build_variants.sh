#!/bin/bash
# Tuning builds of libodegpu with forced kernel-structure policies:
#   scripts/build_variants.sh name:ROLLED:COLD_SHARED:PARAMS_SHARED:MIN_BLOCKS[:BOOK_SHARED] ...  ('-' keeps the model's own)
# -> paper_1810_03931_b200/lib/variants/libodegpu_<name>.so (load with ODEGPU_LIB=...)
set -e
cd "$(dirname "$0")/.."
NVFLAGS="-std=c++20 --expt-relaxed-constexpr -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -Xcompiler -fPIC -Iinclude -Ipaper_1810_03931_b200/csrc"
mkdir -p paper_1810_03931_b200/lib/variants build/variants
for spec in "$@"; do
  IFS=: read name rolled cold params mb book <<< "$spec"
  od=build/variants/$name; mkdir -p $od
  defs=""
  [ "$rolled" != "-" ] && defs="$defs -DODEGPU_POLICY_ROLLED=$rolled"
  [ "$cold" != "-" ] && defs="$defs -DODEGPU_POLICY_COLD_SHARED=$cold"
  [ "$params" != "-" ] && defs="$defs -DODEGPU_POLICY_PARAMS_SHARED=$params"
  [ "$mb" != "-" ] && defs="$defs -DODEGPU_MIN_BLOCKS=$mb"
  [ -n "$book" ] && [ "$book" != "-" ] && defs="$defs -DODEGPU_POLICY_BOOK_SHARED=$book"
  for f in paper_1810_03931_b200/csrc/*.cu; do
    b=$(basename $f .cu)
    nvcc $NVFLAGS $defs -Xptxas -v -c -o $od/$b.o $f 2> $od/$b.ptxas &
  done
  wait
  cat $od/*.ptxas > $od/ptxas.txt
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC -o paper_1810_03931_b200/lib/variants/libodegpu_$name.so $od/*.o
done
