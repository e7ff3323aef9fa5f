#!/bin/bash
# LL: fill idle CTA slots with more chunk groups (new) vs head; auto protocol + parity
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -n 1 gpurun_out/pytest_gpu.log
G='{"scheds":["ag777","ag111","ring","ar822","ar56","ar_ring","a2a"],"sizes":[1024,16384,65536,131072,262144,524288,1048576],"knobs":[{},{"protocol":"ll"}]}'
for i in 1 2; do
SCCL_LIB=$PWD/build/ab/libsccl_exec_head.so timeout 600 python tools/tune.py "$G" > gpurun_out/llf_head_$i.jsonl 2>&1
timeout 600 python tools/tune.py "$G" > gpurun_out/llf_new_$i.jsonl 2>&1
done
