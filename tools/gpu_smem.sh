#!/bin/bash
# shared-memory single-plan kernel: parity tests, single-plan latency per kernel,
# per-phase step cycles, and block-size variants (build/w*.so)
OUT=gpurun_out/${1:-smem1}; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_smem.py -q -x > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 900 python tools/single_plan.py 12 300 1000 1800 > $OUT/single.jsonl 2> $OUT/single.err
for fl in 4 12; do IGP_LIB=build/timing.so timeout 300 python tools/step_timing.py 1000 0.025 32 $fl >> $OUT/timing.txt 2>&1; done
for v in w8 w32; do IGP_LIB=build/$v.so timeout 300 python tools/single_plan.py 300 1000 >> $OUT/variants.jsonl 2>&1; done
echo done > $OUT/DONE
