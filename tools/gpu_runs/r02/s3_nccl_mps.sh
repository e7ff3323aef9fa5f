# round 2 session 3: can NCCL run several ranks on one GPU (plain, and under MPS)?
set -x
timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29591 tools/probes/nccl_dup_probe.py > gpurun_out/s3_nccl_dup_plain.log 2>&1
export CUDA_MPS_PIPE_DIRECTORY=/tmp/mps_pipe CUDA_MPS_LOG_DIRECTORY=/tmp/mps_log
mkdir -p $CUDA_MPS_PIPE_DIRECTORY $CUDA_MPS_LOG_DIRECTORY
nvidia-cuda-mps-control -d; sleep 2
timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29592 tools/probes/nccl_dup_probe.py > gpurun_out/s3_nccl_dup_mps.log 2>&1
echo quit | nvidia-cuda-mps-control
grep -h "RANK\|Duplicate\|rror" gpurun_out/s3_nccl_dup_*.log | head
