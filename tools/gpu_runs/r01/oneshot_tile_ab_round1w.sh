#!/bin/bash
# 16 KiB tiles for one-shot copies up to 512 KiB chunks: same-box A/B + parity
mkdir -p gpurun_out
G='{"scheds":["ag111"],"sizes":[32768,65536,131072,262144,524288,1048576],"knobs":[{},{"protocol":"simple"}]}'
for i in 1 2; do
SCCL_LIB=$PWD/build/ab/libsccl_exec_head.so timeout 600 python tools/tune.py "$G" > gpurun_out/os_head_$i.jsonl 2>&1
timeout 600 python tools/tune.py "$G" > gpurun_out/os_new_$i.jsonl 2>&1
done
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -n 1 gpurun_out/pytest_gpu.log
