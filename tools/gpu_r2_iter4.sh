# sharded compaction + fused offsets scan: tests; C5 bench; E with TPS join vs item join
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sharded.py tests/test_sharding.py tests/test_gpu_parity.py tests/test_gpu_ids.py -m gpu -q -x -p no:cacheprovider > gpurun_out/gputest_iter.log 2>&1
echo "rc=$?" >> gpurun_out/gputest_iter.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/bench_default.log 2>&1
timeout 900 python bench.py --workload E --no-cpu-baseline --no-e2e --steps 5 --warmup 3 --pool 2 > gpurun_out/cfgE_default.log 2>&1
TJ_LIB_PATH=$PWD/paper_1411_3212_b200/_lib/exp_tps0.so timeout 900 python bench.py --workload E --no-cpu-baseline --no-e2e --steps 5 --warmup 3 --pool 2 > gpurun_out/cfgE_tps0.log 2>&1
