mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/gputest_ilp.log 2>&1; echo "rc=$?" >> gpurun_out/gputest_ilp.log
for v in default ilp0 default ilp0; do
  if [ $v = default ]; then unset TJ_LIB_PATH; else export TJ_LIB_PATH=$PWD/paper_1411_3212_b200/_lib/exp_$v.so; fi
  timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline >> gpurun_out/s4_$v.log 2>&1
done
