#!/bin/bash
# balanced chunk groups only for lopsided modulo maps: parity + A/B on the plans that switch
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -n 1 gpurun_out/pytest_gpu.log
G='{"scheds":["a2a","ag777"],"sizes":[131072,524288,2097152,4194304,134217728],"knobs":[{}]}'
for i in 1 2; do
SCCL_LIB=$PWD/build/ab/libsccl_exec_head.so timeout 600 python tools/tune.py "$G" > gpurun_out/grp3_head_$i.jsonl 2>&1
timeout 600 python tools/tune.py "$G" > gpurun_out/grp3_new_$i.jsonl 2>&1
done
