mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
for W in ${WLS:-A B C5 C10 C20}; do
  timeout 900 python bench.py --workload $W --no-cpu-baseline --no-e2e --steps 5 --pool 2 > gpurun_out/bench_$W.log 2>&1; echo $W=$?
  tail -1 gpurun_out/bench_$W.log | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['config']['workload'],d['value'],d['p50_tick_ms'],d['config']['results_per_tick'],d['stage_ms'])" 2>/dev/null
done
