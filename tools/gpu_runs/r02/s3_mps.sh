# round 2 session 3: the one-rank-per-process path with 8 processes CONCURRENT on one GPU under MPS (not time-sliced): bench N>1 code path timed
set -x
make -s -j8 all > /dev/null
export CUDA_MPS_PIPE_DIRECTORY=/tmp/mps_pipe CUDA_MPS_LOG_DIRECTORY=/tmp/mps_log
mkdir -p $CUDA_MPS_PIPE_DIRECTORY $CUDA_MPS_LOG_DIRECTORY
nvidia-cuda-mps-control -d
sleep 2
SCCL_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29561 bench.py --gpus 8 --steps 10 --warmup 3 --bytes 16777216 --no-sweep > gpurun_out/s3_mps_share8_16m.log 2>&1
SCCL_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29562 bench.py --gpus 8 --steps 10 --warmup 3 --bytes 134217728 --no-sweep > gpurun_out/s3_mps_share8_128m.log 2>&1
echo quit | nvidia-cuda-mps-control
sleep 1
cat $CUDA_MPS_LOG_DIRECTORY/control.log | tail -5
for f in gpurun_out/s3_mps_share8_*.log; do grep -h '^{' $f | cut -c1-300; tail -3 $f; done
