# round 2 session 3: bench N>1 path with the CTA-count autotune: one-rank NCCL self-test and shared-GPU worlds 2 and 8
set -x
make -s -j8 all > /dev/null
SCCL_BENCH_FORCE_MULTI=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 1 --steps 5 --warmup 3 --bytes 16777216 > gpurun_out/s3_multi2_world1.log 2>&1
SCCL_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --bytes 16777216 > gpurun_out/s3_multi2_share2.log 2>&1
SCCL_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 8 --steps 3 --warmup 3 --bytes 4194304 > gpurun_out/s3_multi2_share8.log 2>&1
for f in gpurun_out/s3_multi2_*.log; do grep -h '^{' $f | cut -c1-200; done
