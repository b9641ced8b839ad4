# sort-branch / scatter contention sweep: fused x/y gather; scatter CTAs per SM
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/gputest_sweep.log 2>&1; echo "rc=$?" >> gpurun_out/gputest_sweep.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/sw_default.log 2>&1
TJ_LIB_PATH=$PWD/paper_1411_3212_b200/_lib/exp_gxy.so timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/sw_gxy.log 2>&1
TJ_LIB_PATH=$PWD/paper_1411_3212_b200/_lib/exp_even.so timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/sw_even.log 2>&1
for P in 2 4 6 12; do TJ_SCATTER_PER_SM=$P timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/sw_sps$P.log 2>&1; done
TJ_SIDE_PRIO=1 timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/sw_prio.log 2>&1
