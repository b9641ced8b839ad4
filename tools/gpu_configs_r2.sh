# every BASELINE configuration that fits one GPU on the current build (5 timed ticks each)
mkdir -p gpurun_out
for W in ${WLS:-A B C2 C5 C10 C20 E}; do
  timeout 900 python bench.py --workload $W --no-cpu-baseline --no-e2e --steps 5 --warmup 3 --pool 2 > gpurun_out/cfg_$W.log 2>&1; echo "$W rc=$?"
done
