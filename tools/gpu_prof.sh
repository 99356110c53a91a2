#!/bin/bash
# ncu --set full of the second k_place launch at a given config.  usage: tools/gpu_prof.sh tag S m flags [lib]
TAG=$1; S=${2:-2368}; M=${3:-10000}; FL=${4:-0}
OUT=gpurun_out/$TAG; mkdir -p $OUT
[ -n "$5" ] && export IGP_LIB=$5
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_place -s 1 -c 1 \
  -o $OUT/place python tools/profile_place.py $S $M $FL > $OUT/ncu_full.log 2>&1
tail -3 $OUT/ncu_full.log
