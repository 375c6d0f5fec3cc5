#!/bin/bash
# A/B builds: the default objects (make lib) with selected translation units
# recompiled under extra flags.
#   TUS="models_duffing models_valve" scripts/build_flag_variants.sh name:"-DFOO=1 -DBAR=2" ...
# -> paper_1810_03931_b200/lib/variants/libodegpu_<name>.so (ODEGPU_LIB=... to load)
set -e
cd "$(dirname "$0")/.."
make -s lib
NVFLAGS="-std=c++20 --expt-relaxed-constexpr -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -Xcompiler -fPIC -Iinclude -Ipaper_1810_03931_b200/csrc"
TUS=${TUS:-"models_duffing models_valve"}
mkdir -p paper_1810_03931_b200/lib/variants
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  od=build/variants/$name; rm -rf $od; mkdir -p $od
  cp build/obj/*.o $od/
  for tu in $TUS; do
    nvcc $NVFLAGS $flags -Xptxas -v -c -o $od/$tu.o paper_1810_03931_b200/csrc/$tu.cu 2> $od/$tu.ptxas &
  done
  wait
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC -o paper_1810_03931_b200/lib/variants/libodegpu_$name.so $od/*.o
  echo "built $name ($flags)"
done
