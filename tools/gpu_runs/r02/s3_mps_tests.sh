# round 2 session 3: multi-process GPU tests with the ranks running CONCURRENTLY under MPS (8-process multi-device harness IPC+VMM with bursts; LL parity test)
set -x
make -s -j8 all > /dev/null
export CUDA_MPS_PIPE_DIRECTORY=/tmp/mps_pipe CUDA_MPS_LOG_DIRECTORY=/tmp/mps_log
mkdir -p $CUDA_MPS_PIPE_DIRECTORY $CUDA_MPS_LOG_DIRECTORY
nvidia-cuda-mps-control -d
sleep 2
SCCL_MULTIDEVICE_SHARE=1 SCCL_MULTIDEVICE_WORLD=8 SCCL_MULTIDEVICE_NCH=16 timeout 1700 python -m pytest tests/test_gpu_multidevice.py -x -q -k one_rank -rs > gpurun_out/s3_mps_multidev8.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_ll_parity.py -x -q > gpurun_out/s3_mps_llparity.log 2>&1
echo quit | nvidia-cuda-mps-control
tail -3 gpurun_out/s3_mps_multidev8.log; tail -3 gpurun_out/s3_mps_llparity.log
