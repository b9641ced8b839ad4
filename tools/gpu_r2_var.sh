# variant comparison (TJ_LIB_PATH) + launch list of the shuffled-id tick
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_ids.py tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/gputest_var.log 2>&1
echo "rc=$?" >> gpurun_out/gputest_var.log
for v in ${VARIANTS:-default l0nopad l0pad}; do
  if [ $v = default ]; then unset TJ_LIB_PATH; else export TJ_LIB_PATH=$PWD/paper_1411_3212_b200/_lib/exp_$v.so; fi
  timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/bench_$v.log 2>&1; echo "rc=$?" >> gpurun_out/bench_$v.log
done
unset TJ_LIB_PATH
timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --shuffle-ids > gpurun_out/bench_shuffled.log 2>&1; echo "rc=$?" >> gpurun_out/bench_shuffled.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 500 --csv --log-file gpurun_out/launches_shuf.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --shuffle-ids > gpurun_out/ncu_shuf.log 2>&1
