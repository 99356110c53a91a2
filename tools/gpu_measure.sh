#!/bin/bash
# Config sweep + headline bench line.  usage: tools/gpu_measure.sh tag [configs...]
OUT=gpurun_out/$1; shift; mkdir -p $OUT
timeout 1500 python tools/bench_configs.py "$@" > $OUT/configs.jsonl 2> $OUT/configs.err; echo "configs rc=$?" >> $OUT/configs.err
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
cat $OUT/configs.jsonl $OUT/bench.json; tail -3 $OUT/configs.err $OUT/bench.err
