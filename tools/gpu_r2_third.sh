# round 2 (session 3): GPU tests incl. full-size parity, bench (our arm), reference arm, launch list
nproc > gpurun_out/nproc.txt; free -g >> gpurun_out/nproc.txt
timeout 2700 python -m pytest tests -m gpu -q --durations=25 -p no:cacheprovider > gpurun_out/gputest.log 2>&1
echo "rc=$?" >> gpurun_out/gputest.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "rc=$?" >> gpurun_out/bench.log
timeout 1200 python bench.py --impl reference --steps 6 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/bench_ref.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_b.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_b.log
