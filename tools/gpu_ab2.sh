#!/bin/bash
# A/B timing only: pairs "variant@S,m,flags" (IGP_LIB=build/<variant>.so).  usage: tools/gpu_ab2.sh tag pair...
OUT=gpurun_out/$1; shift; mkdir -p $OUT
for p in "$@"; do v=${p%%@*}; c=${p#*@}; IGP_LIB=build/$v.so timeout 900 python tools/quick_time.py $c >> $OUT/ab.log 2>&1; done
