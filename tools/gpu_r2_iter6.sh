mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ids.py -m gpu -q -x -p no:cacheprovider > gpurun_out/gputest_iter.log 2>&1
echo "rc=$?" >> gpurun_out/gputest_iter.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/bench_default.log 2>&1
for W in C20 C10 B; do timeout 900 python bench.py --workload $W --no-cpu-baseline --no-e2e --steps 5 --warmup 3 --pool 2 > gpurun_out/cfg_$W.log 2>&1; done
