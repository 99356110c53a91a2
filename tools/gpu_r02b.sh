OUT=gpurun_out/r02_b; mkdir -p $OUT
timeout 600 python tools/host_chunks.py 2368 1 2 4 > $OUT/chunks.txt 2>&1
timeout 1200 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
