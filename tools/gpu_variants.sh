#!/bin/bash
# A/B of library build variants (build/<name>.so) at one batch wave each.
# usage: gpurun -- bash tools/gpu_variants.sh TAG name [name ...]
TAG=$1; shift; OUT=gpurun_out/$TAG; mkdir -p $OUT
for v in "$@"; do
  IGP_LIB=build/$v.so timeout 600 python tools/quick_time.py 0,10000,0 0,1000,0 >> $OUT/variants.txt 2>&1
done
