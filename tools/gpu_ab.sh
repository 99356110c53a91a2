#!/bin/bash
# parity tests + A/B timing of library variants in build/.  usage: tools/gpu_ab.sh tag "v1 v2 ..." "S,m,flags ..."
OUT=gpurun_out/${1:-ab}; mkdir -p $OUT
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
for v in ${2:-s4m4}; do IGP_LIB=build/$v.so timeout 600 python tools/quick_time.py ${3:-2368,10000,0} >> $OUT/ab.log 2>&1; done
