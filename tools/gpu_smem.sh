#!/bin/bash
# shared-memory single-plan kernel: parity tests, single-plan latency per kernel,
# per-phase step cycles (build/timing.so = -DIGP_TIMING=1)
OUT=gpurun_out/${1:-smem1}; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_smem.py -q -x > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 900 python tools/single_plan.py 12 300 1000 1200 > $OUT/single.jsonl 2> $OUT/single.err
IGP_LIB=build/timing.so timeout 300 python tools/step_timing.py 1000 0.025 32 12 >> $OUT/timing.txt 2>&1
echo done > $OUT/DONE
