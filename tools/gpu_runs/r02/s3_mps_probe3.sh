# round 2 session 3: MPS probe (8 concurrent processes on one GPU) repeated 3 times for medians: LL parity vs entry handshake, simple sizes
set -x
make -s -j8 all > /dev/null
export CUDA_MPS_PIPE_DIRECTORY=/tmp/mps_pipe CUDA_MPS_LOG_DIRECTORY=/tmp/mps_log
mkdir -p $CUDA_MPS_PIPE_DIRECTORY $CUDA_MPS_LOG_DIRECTORY
nvidia-cuda-mps-control -d
sleep 2
for rep in 1 2 3; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 2958$rep tools/probes/mps_multiproc.py >> gpurun_out/s3_mps_probe8x3.jsonl 2>> gpurun_out/s3_mps_probe8x3.err
done
echo quit | nvidia-cuda-mps-control
wc -l gpurun_out/s3_mps_probe8x3.jsonl
