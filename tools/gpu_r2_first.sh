nproc > gpurun_out/nproc.txt; free -g >> gpurun_out/nproc.txt; nvidia-smi >> gpurun_out/nproc.txt
timeout 2400 python -m pytest tests -m gpu -q --durations=30 -p no:cacheprovider > gpurun_out/gputest.log 2>&1
echo "rc=$?" >> gpurun_out/gputest.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1
echo "rc=$?" >> gpurun_out/bench.log
