# iteration: parity subset + bench + ncu --set full of the decode (id mode 0)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ids.py tests/test_gpu_sharded.py tests/test_gpu_ug.py -m gpu -q -x -p no:cacheprovider > gpurun_out/gputest_iter.log 2>&1
echo "rc=$?" >> gpurun_out/gputest_iter.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_iter.log 2>&1; echo "rc=$?" >> gpurun_out/bench_iter.log
timeout 900 ncu --set full --clock-control none --import-source on -k k_decode_query --launch-skip 9 -c 1 -o gpurun_out/prof_dec python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/prof_dec.log 2>&1
echo ncu=$? >> gpurun_out/prof_dec.log
