OUT=gpurun_out/r02_d; mkdir -p $OUT
timeout 1500 python -m pytest tests -q -m gpu --durations=25 > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python tools/c5_stream.py 1000000 4096 --check 24576 > $OUT/c5_1m.json 2> $OUT/c5_1m.err
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
echo done > $OUT/DONE
