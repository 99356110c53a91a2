#!/bin/bash
# A/B of prefetch variants: timing + DRAM bytes of one headline k_place launch.  usage: tools/gpu_pf.sh tag v1 v2 ...
OUT=gpurun_out/$1; shift; mkdir -p $OUT
for rep in 1 2; do for v in "$@"; do IGP_LIB=build/$v.so timeout 900 python tools/quick_time.py 2368,10000,0 4096,1000,0 >> $OUT/ab.log 2>&1; done; done
for v in "$@"; do
  IGP_LIB=build/$v.so timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct \
    --clock-control none -k regex:k_place -s 1 -c 1 --csv python tools/profile_place.py 2368 10000 0 > $OUT/dram_$v.csv 2>&1
done
cat $OUT/ab.log; for v in "$@"; do echo "== $v"; grep -E "dram__|hit_rate" $OUT/dram_$v.csv | awk -F'","' '{print $(NF-2), $NF}'; done
