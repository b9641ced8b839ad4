# round-2 evidence on the current build: launch list, ncu --set full of the tick's main kernels,
# the reference engine's CPU timings on A and B (n_workers 1 and all host cores)
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_r2.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/launches_r2_bench.log 2>&1
echo ncu_list=$? >> gpurun_out/launches_r2_bench.log
timeout 1500 ncu --set full --clock-control none --import-source on -k "regex:k_mbr|k_codes|k_radix_downsweep|k_gather|k_query_count|k_query_fill|k_join|k_decode_query<0>" --launch-skip 30 -c 10 -o gpurun_out/prof_r2c python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/prof_r2c.log 2>&1
echo ncu_full=$? >> gpurun_out/prof_r2c.log
timeout 2400 python tools/ref_cpu_timings.py --b-ticks 3 > gpurun_out/ref_cpu.json 2> gpurun_out/ref_cpu.log; echo "rc=$?" >> gpurun_out/ref_cpu.log
