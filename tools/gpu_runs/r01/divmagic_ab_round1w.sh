#!/bin/bash
# same-box A/B: byte-part split by magic reciprocal + 32-bit tile counts (new) vs 64-bit divides (head)
set -x
mkdir -p gpurun_out
G='{"scheds":["ag777","ring","ar56","ar_ring","ar822","a2a"],"sizes":[1024,65536,1048576,16777216,134217728],"knobs":[{}]}'
for i in 1 2; do
SCCL_LIB=$PWD/build/ab/libsccl_exec_head.so timeout 600 python tools/tune.py "$G" > gpurun_out/divm_head_$i.jsonl 2>&1
timeout 600 python tools/tune.py "$G" > gpurun_out/divm_new_$i.jsonl 2>&1
done
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
