mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sharded.py tests/test_sharding.py tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/gputest_iter.log 2>&1
echo "rc=$?" >> gpurun_out/gputest_iter.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/bench_default.log 2>&1
timeout 900 python bench.py --workload C20 --no-cpu-baseline --no-e2e --steps 5 --warmup 3 --pool 2 > gpurun_out/cfg_C20.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --sharded > gpurun_out/bench_sharded1.log 2>&1
timeout 600 python tools/sanitize_r2.py > gpurun_out/sanitize_plain.log 2>&1; echo rc=$? >> gpurun_out/sanitize_plain.log
timeout 1200 compute-sanitizer --tool memcheck python tools/sanitize_r2.py > gpurun_out/sanitize_memcheck.log 2>&1; echo rc=$? >> gpurun_out/sanitize_memcheck.log
