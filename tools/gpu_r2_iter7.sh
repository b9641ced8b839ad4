mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ids.py -m gpu -q -x -p no:cacheprovider > gpurun_out/gputest_iter.log 2>&1
echo "rc=$?" >> gpurun_out/gputest_iter.log
for v in default gtmp smem8; do
  if [ $v = default ]; then unset TJ_LIB_PATH; else export TJ_LIB_PATH=$PWD/paper_1411_3212_b200/_lib/exp_$v.so; fi
  timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/bench_$v.log 2>&1
  timeout 900 python bench.py --workload C20 --no-cpu-baseline --no-e2e --steps 5 --warmup 3 --pool 2 > gpurun_out/c20_$v.log 2>&1
done
