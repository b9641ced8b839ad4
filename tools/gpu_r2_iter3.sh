# iteration: parity subset + bench default vs variants (VARIANTS)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ids.py tests/test_gpu_ug.py -m gpu -q -x -p no:cacheprovider > gpurun_out/gputest_iter.log 2>&1
echo "rc=$?" >> gpurun_out/gputest_iter.log
for v in ${VARIANTS:-default}; do
  if [ $v = default ]; then unset TJ_LIB_PATH; else export TJ_LIB_PATH=$PWD/paper_1411_3212_b200/_lib/exp_$v.so; fi
  timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/bench_$v.log 2>&1; echo "rc=$?" >> gpurun_out/bench_$v.log
done
