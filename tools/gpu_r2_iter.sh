# quick iteration: parity subset + bench + sharded bench (N=1 NCCL, torchrun)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ids.py tests/test_gpu_sharded.py tests/test_gpu_ug.py -m gpu -q -x -p no:cacheprovider > gpurun_out/gputest_iter.log 2>&1
echo "rc=$?" >> gpurun_out/gputest_iter.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_iter.log 2>&1; echo "rc=$?" >> gpurun_out/bench_iter.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --sharded > gpurun_out/bench_sharded1.log 2>&1; echo "rc=$?" >> gpurun_out/bench_sharded1.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 10 --warmup 3 --no-cpu-baseline --sharded > gpurun_out/bench_sharded_trun.log 2>&1; echo "rc=$?" >> gpurun_out/bench_sharded_trun.log
