#!/bin/bash
# same-box A/B: compute warps skip copy-only programs, no chunk-group modulo per op (new) vs head
set -x
mkdir -p gpurun_out
G='{"scheds":["ag777","ring","ag111","a2a","ar56"],"sizes":[262144,1048576,4194304,16777216,134217728],"knobs":[{}]}'
for i in 1 2; do
SCCL_LIB=$PWD/build/ab/libsccl_exec_head.so timeout 600 python tools/tune.py "$G" > gpurun_out/idle_head_$i.jsonl 2>&1
timeout 600 python tools/tune.py "$G" > gpurun_out/idle_new_$i.jsonl 2>&1
done
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
