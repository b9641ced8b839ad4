bash tools/gpu_iter.sh
LIBS="libtickjoin_b200.so exp_mb8.so exp_mb12.so" bash tools/gpu_variants.sh
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/launches_bench.log 2>&1
