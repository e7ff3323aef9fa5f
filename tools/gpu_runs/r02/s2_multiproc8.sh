# round 2 session 2: the one-rank-per-GPU harness with 8 processes time-sliced on cuda:0 (IPC and VMM):
# every P=8 schedule the bench uses, incl. (7,7,7) and (56,14,14), across 8 separate contexts
SCCL_MULTIDEVICE_SHARE=1 SCCL_MULTIDEVICE_WORLD=8 timeout 3000 python -m pytest tests/test_gpu_multidevice.py -x -q -rs > gpurun_out/s2_multiproc8.log 2>&1
tail -5 gpurun_out/s2_multiproc8.log
