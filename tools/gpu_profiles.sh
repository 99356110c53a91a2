#!/bin/bash
# Round evidence: ncu launch list of the bench command, full ncu capture of k_place at the
# bench configuration and of k_solo_grid at C3.  usage: tools/gpu_profiles.sh tag
OUT=gpurun_out/$1; mkdir -p $OUT
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/ncu_bench.log 2>&1
echo "launch list rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_solo_grid -c 1 \
  -o $OUT/grid python tools/bench_configs.py c3grid > $OUT/ncu_grid.log 2>&1
echo "grid rc=$?"
timeout 2400 ncu --set full --clock-control none --import-source on -k regex:k_place -s 1 -c 1 \
  -o $OUT/place python tools/profile_place.py 2368 10000 0 > $OUT/ncu_place.log 2>&1
echo "place rc=$?"
