#!/bin/bash
# fast-kernel pass: its parity tests, an A/B against the exact kernel, the full GPU suite
OUT=gpurun_out/${1:-fast1}; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_fast.py -q -x > $OUT/pytest_fast.log 2>&1; echo "rc=$?" >> $OUT/pytest_fast.log
for rep in 1 2; do
  timeout 600 python tools/quick_time.py 0,10000,0 0,10000,536870912 0,1000,0 0,1000,536870912 >> $OUT/ab.txt 2>&1
done
timeout 1500 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
echo done > $OUT/DONE
