# Parity + bench of experimental library variants against the default build.
#   bash tools/build_variant.sh st768 -DTJ_DQ_STAGE=768       # here, once per variant
#   gpurun -- 'VARIANTS="default st768" WLS="C5 C20" bash tools/gpu_variant_sweep.sh'
# PARITY=<variant>: run the parity suite on that variant first.
mkdir -p gpurun_out
if [ -n "$PARITY" ]; then
  TJ_LIB_PATH=$PWD/paper_1411_3212_b200/_lib/exp_$PARITY.so timeout 900 python -m pytest tests/test_gpu_parity.py \
    tests/test_gpu_ids.py -m gpu -q -x -p no:cacheprovider > gpurun_out/sweep_parity_$PARITY.log 2>&1
  echo "rc=$?" >> gpurun_out/sweep_parity_$PARITY.log
fi
for w in ${WLS:-C5}; do
  for v in ${VARIANTS:-default}; do
    if [ $v = default ]; then unset TJ_LIB_PATH; else export TJ_LIB_PATH=$PWD/paper_1411_3212_b200/_lib/exp_$v.so; fi
    timeout 900 python bench.py --workload $w --steps ${STEPS:-20} --warmup 5 --no-e2e --no-cpu-baseline \
      >> gpurun_out/sweep_${w}_$v.log 2>&1
    echo "rc=$?" >> gpurun_out/sweep_${w}_$v.log
  done
done
