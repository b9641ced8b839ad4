# round-2 final evidence on the committed build: the driver's bench command, the reference arm,
# full GPU suite, smoke, launch list and ncu --set full of the tick's main kernels
mkdir -p gpurun_out
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/final_bench.log 2>&1; echo "rc=$?" >> gpurun_out/final_bench.log
timeout 600 python bench.py --shuffle-ids --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/final_bench_shuffled.log 2>&1
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final_gputest.log 2>&1; echo "rc=$?" >> gpurun_out/final_gputest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/final_smoke.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 700 --csv --log-file gpurun_out/final_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k "regex:k_mbr|k_codes|k_radix_downsweep|k_gather|k_query_count|k_query_fill|k_join" --launch-skip 24 -c 8 -o gpurun_out/final_prof python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/final_prof.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k k_decode_query --launch-skip 9 -c 1 -o gpurun_out/final_prof_dec python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/final_prof_dec.log 2>&1
