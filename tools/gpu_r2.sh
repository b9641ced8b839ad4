mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo bench=$?; tail -1 gpurun_out/bench.log | cut -c1-3000
TJ_NO_GRAPH=1 timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_nograph.log 2>&1; echo nograph=$?; tail -1 gpurun_out/bench_nograph.log | cut -c1-300
timeout 600 python bench.py --no-cpu-baseline --sharded > gpurun_out/bench_sharded.log 2>&1; echo sharded=$?; tail -3 gpurun_out/bench_sharded.log | cut -c1-3000
timeout 600 python bench.py --no-cpu-baseline --workload A --steps 20 > gpurun_out/bench_A.log 2>&1; echo A=$?; tail -1 gpurun_out/bench_A.log | cut -c1-600
TJ_NO_GRAPH=1 timeout 600 python bench.py --no-cpu-baseline --workload A --steps 20 --no-e2e > gpurun_out/bench_A_nograph.log 2>&1; echo Ang=$?; tail -1 gpurun_out/bench_A_nograph.log | cut -c1-300
