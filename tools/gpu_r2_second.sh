# round 2: GPU tests (incl. full-size parity), bench (our arm), reference arm, reference CPU timings
timeout 2400 python -m pytest tests -m gpu -q --durations=15 -p no:cacheprovider > gpurun_out/gputest.log 2>&1
echo "rc=$?" >> gpurun_out/gputest.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "rc=$?" >> gpurun_out/bench.log
timeout 1200 python bench.py --impl reference --steps 6 --warmup 2 > gpurun_out/bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/bench_ref.log
timeout 1800 python tools/ref_cpu_timings.py --b-ticks 3 > gpurun_out/ref_cpu.json 2> gpurun_out/ref_cpu.log; echo "rc=$?" >> gpurun_out/ref_cpu.log
