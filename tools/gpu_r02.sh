#!/bin/bash
# Round-2 GPU pass: full GPU suite and smoke (unless skip-tests), the bench line
# and the reference arm, a two-wave batch, the config sweep, the ncu launch list
# and one --set full capture of k_place at the bench batch.
# usage: gpurun -- bash tools/gpu_r02.sh TAG [skip-tests]
TAG=${1:-r02}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/gpu.txt 2>&1
lscpu | head -20 > $OUT/cpu.txt
if [ "$2" != "skip-tests" ]; then
  timeout 1500 python -m pytest tests -q -m gpu --durations=25 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
fi
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
timeout 1200 python bench.py --scenarios 5920 --steps 3 --warmup 3 --check 4 --no-cpu-baseline > $OUT/bench_2wave.json 2> $OUT/bench_2wave.err
timeout 1500 python tools/bench_configs.py > $OUT/configs.jsonl 2> $OUT/configs.err; echo "configs rc=$?" >> $OUT/configs.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --check 0 > $OUT/ncu_bench.log 2>&1
timeout 2400 ncu --set full --clock-control none --import-source on -k regex:k_place -s 1 -c 1 \
  -o $OUT/place python tools/profile_place.py 0 10000 0 > $OUT/ncu_full.log 2>&1
echo done > $OUT/DONE
