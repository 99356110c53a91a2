#!/bin/bash
# Build A/B variants of the library into build/ (select one with IGP_LIB=build/<name>.so).
# usage: tools/build_variants.sh name:"-DFLAG=.. -DFLAG2=.." [...]
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC -shared"
SRC=paper_2211_01713_b200/csrc/igniter_kernels.cu
mkdir -p build
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  $NV $flags -o build/$name.so $SRC 2>&1 | grep -E "error" &
done
wait
ls -la build/
