#!/bin/bash
# 16 KiB tiles for wide reductions with chunks <= 256 KiB: same-box A/B (auto protocol) + parity
mkdir -p gpurun_out
G='{"scheds":["ar822"],"sizes":[262144,524288,1048576,2097152,4194304],"knobs":[{},{"protocol":"simple"}]}'
for i in 1 2; do
SCCL_LIB=$PWD/build/ab/libsccl_exec_head.so timeout 600 python tools/tune.py "$G" > gpurun_out/wide_head_$i.jsonl 2>&1
timeout 600 python tools/tune.py "$G" > gpurun_out/wide_new_$i.jsonl 2>&1
done
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -n 1 gpurun_out/pytest_gpu.log
