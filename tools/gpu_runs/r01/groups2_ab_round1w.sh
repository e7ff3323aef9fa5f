#!/bin/bash
# balanced chunk groups only when 3 % better balanced (new) vs chunk % kc (head): parity + A/B
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -n 1 gpurun_out/pytest_gpu.log
G='{"scheds":["a2a","ag777","ar56"],"sizes":[4194304,16777216,134217728],"knobs":[{}]}'
for i in 1 2; do
SCCL_LIB=$PWD/build/ab/libsccl_exec_head.so timeout 600 python tools/tune.py "$G" > gpurun_out/grp2_head_$i.jsonl 2>&1
timeout 600 python tools/tune.py "$G" > gpurun_out/grp2_new_$i.jsonl 2>&1
done
