#!/bin/bash
# One GPU-box pass: parity tests, smoke, bench line, ncu launch list + full capture of k_place.
# usage (from this container): gpurun --timeout 2400 -- bash tools/gpu_check.sh [tag]
TAG=${1:-r01}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/gpu.txt 2>&1
lscpu | head -20 > $OUT/cpu.txt; nproc >> $OUT/cpu.txt
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --scenarios 592 > $OUT/ncu_bench.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_place -s 1 -c 1 \
  -o $OUT/place python tools/profile_place.py 592 10000 0 > $OUT/ncu_full.log 2>&1
echo done > $OUT/DONE
