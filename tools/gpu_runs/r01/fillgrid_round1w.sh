#!/bin/bash
# bulk plans: trade byte parts for chunk groups when that fills >= 25 % more CTA slots (new) vs head
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -n 1 gpurun_out/pytest_gpu.log
G='{"scheds":["ag777","ag111","ring","ar822","ar56","ar_ring","a2a"],"sizes":[524288,1048576,2097152,4194304,8388608,16777216,67108864,134217728],"knobs":[{}]}'
for i in 1 2; do
SCCL_LIB=$PWD/build/ab/libsccl_exec_head.so timeout 600 python tools/tune.py "$G" > gpurun_out/fg_head_$i.jsonl 2>&1
timeout 600 python tools/tune.py "$G" > gpurun_out/fg_new_$i.jsonl 2>&1
done
