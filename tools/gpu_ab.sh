#!/bin/bash
# A/B of library variants (build/<name>.so), interleaved twice, plus the GPU
# parity tests on the default in-tree build.
# usage: gpurun -- bash tools/gpu_ab.sh TAG "pytest -k expression" name [name ...]
TAG=$1; K=$2; shift 2; OUT=gpurun_out/$TAG; mkdir -p $OUT
if [ -n "$K" ]; then
  timeout 900 python -m pytest tests -q -m gpu -x -k "$K" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
fi
for rep in 1 2; do
  for v in "$@"; do
    IGP_LIB=build/$v.so timeout 600 python tools/quick_time.py 0,10000,0 0,1000,0 >> $OUT/variants.txt 2>&1
  done
done
echo done > $OUT/DONE
