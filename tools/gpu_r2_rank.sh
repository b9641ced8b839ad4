# rank mode (non-monotone ids): GPU tests, bench arange vs shuffled ids, ncu source-level captures
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ids.py tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/gputest_ids.log 2>&1
echo "rc=$?" >> gpurun_out/gputest_ids.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/bench_arange.log 2>&1; echo "rc=$?" >> gpurun_out/bench_arange.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --shuffle-ids > gpurun_out/bench_shuffled.log 2>&1; echo "rc=$?" >> gpurun_out/bench_shuffled.log
KREGEX="k_decode_query|k_join|k_query_fill|k_query_count" SKIP=16 COUNT=4 OUT=prof_r2 bash tools/gpu_prof.sh
