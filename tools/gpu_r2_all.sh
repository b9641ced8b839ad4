# full GPU suite + bench (default) + sharded bench at N=1 (NCCL one rank, tj_tick_sharded)
mkdir -p gpurun_out
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > gpurun_out/gputest_all.log 2>&1
echo "rc=$?" >> gpurun_out/gputest_all.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_all.log 2>&1; echo "rc=$?" >> gpurun_out/bench_all.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --sharded > gpurun_out/bench_sharded1.log 2>&1; echo "rc=$?" >> gpurun_out/bench_sharded1.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 10 --warmup 3 --no-cpu-baseline --sharded > gpurun_out/bench_sharded_trun.log 2>&1; echo "rc=$?" >> gpurun_out/bench_sharded_trun.log
