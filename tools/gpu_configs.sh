# every BASELINE config that fits one GPU: A, B, C at 2/5/10/20u, E (50M)
mkdir -p gpurun_out
for W in A B C2 C5 C10 C20; do
  timeout 900 python bench.py --workload $W --no-cpu-baseline --no-e2e --steps 5 --pool 2 > gpurun_out/bench_$W.log 2>&1; echo $W=$?
  tail -1 gpurun_out/bench_$W.log | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['config']['workload'],d['value'],d['p50_tick_ms'],d['config']['results_per_tick'],d['stage_ms'])" 2>/dev/null
done
timeout 1500 python bench.py --workload E --no-cpu-baseline --no-e2e --steps 3 --warmup 3 --pool 1 > gpurun_out/bench_E.log 2>&1; echo E=$?
tail -3 gpurun_out/bench_E.log | cut -c1-1500
