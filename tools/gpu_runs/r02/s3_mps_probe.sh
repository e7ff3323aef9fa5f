# round 2 session 3: one-rank-per-process path timed with 8 (and 2) processes concurrent on one GPU under MPS: LL parity vs handshake, simple sizes
set -x
make -s -j8 all > /dev/null
export CUDA_MPS_PIPE_DIRECTORY=/tmp/mps_pipe CUDA_MPS_LOG_DIRECTORY=/tmp/mps_log
mkdir -p $CUDA_MPS_PIPE_DIRECTORY $CUDA_MPS_LOG_DIRECTORY
nvidia-cuda-mps-control -d
sleep 2
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29571 tools/probes/mps_multiproc.py > gpurun_out/s3_mps_probe8.jsonl 2> gpurun_out/s3_mps_probe8.err

echo quit | nvidia-cuda-mps-control
cat gpurun_out/s3_mps_probe8.jsonl
