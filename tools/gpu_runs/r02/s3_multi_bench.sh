# round 2 session 3: the bench N>1 path after the section/agreement rework:
# one-rank NCCL self-test (every comparison section) and shared-GPU worlds 2 and 8 (gloo)
set -x
make -s -j8 all > /dev/null
SCCL_BENCH_FORCE_MULTI=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 1 --steps 5 --warmup 3 --bytes 16777216 > gpurun_out/s3_multi_world1.log 2>&1
SCCL_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --bytes 16777216 > gpurun_out/s3_share2.log 2>&1
SCCL_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 8 --steps 3 --warmup 3 --bytes 4194304 > gpurun_out/s3_share8.log 2>&1
timeout 600 python -m pytest tests/test_gpu_multiprocess.py tests/test_gpu_nvls.py tests/test_gpu_watchdog.py -x -q -rs > gpurun_out/s3_multiproc_tests.log 2>&1
tail -c 1500 gpurun_out/s3_multi_world1.log; tail -3 gpurun_out/s3_multiproc_tests.log
