mkdir -p gpurun_out
for v in default match rpl8 tmq6 tmq24; do
  if [ $v = default ]; then unset TJ_LIB_PATH; else export TJ_LIB_PATH=$PWD/paper_1411_3212_b200/_lib/exp_$v.so; fi
  timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/s2_$v.log 2>&1
done
unset TJ_LIB_PATH
TJ_LIB_PATH=$PWD/paper_1411_3212_b200/_lib/exp_match.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/gputest_match.log 2>&1; echo "rc=$?" >> gpurun_out/gputest_match.log
