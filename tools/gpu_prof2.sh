# parity iteration + launch list + ncu --set full of the tick's main kernels
bash tools/gpu_iter.sh
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/launches_bench.log 2>&1
echo ncu_list=$?
KREGEX="k_decode_query|k_join|k_query_fill|k_query_count|k_radix_downsweep|k_radix_upsweep" SKIP=24 COUNT=8 OUT=prof_main bash tools/gpu_prof.sh
