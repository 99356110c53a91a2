#!/bin/bash
# Run arbitrary commands on the GPU box, logging to gpurun_out/<tag>/out.log.  usage: tools/gpu_cmd.sh tag 'cmd1' 'cmd2' ...
OUT=gpurun_out/$1; shift; mkdir -p $OUT
for c in "$@"; do echo "### $c" >> $OUT/out.log; timeout 1200 bash -c "$c" >> $OUT/out.log 2>&1; echo "rc=$?" >> $OUT/out.log; done
cat $OUT/out.log
