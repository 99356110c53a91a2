OUT=gpurun_out/r02_c; mkdir -p $OUT
timeout 600 python tools/host_chunks.py 2368 1 2 4 > $OUT/chunks.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_stream.py tests/test_gpu_multi.py tests/ref_suite tests/test_boundary.py tests/test_ref_headline.py -q -m gpu > $OUT/pytest_new.log 2>&1; echo "rc=$?" >> $OUT/pytest_new.log
timeout 600 python tools/c5_stream.py 200000 4096 --check 24576 > $OUT/c5_200k.json 2> $OUT/c5_200k.err
timeout 300 env COOP_FROM=100000000 python tools/c5_stream.py 100000 4096 > $OUT/c5_100k_cta.json 2> $OUT/c5_100k_cta.err
echo done > $OUT/DONE
