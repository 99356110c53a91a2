#!/bin/bash
# GPU parity suite (optionally a subset).  usage: tools/gpu_tests.sh tag [pytest args...]
OUT=gpurun_out/$1; shift; mkdir -p $OUT
timeout 1800 python -m pytest tests -q -m gpu --durations=15 "$@" > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
tail -25 $OUT/pytest_gpu.log
