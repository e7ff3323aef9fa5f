#!/bin/bash
# LL: grow byte parts when chunk groups are exhausted (new) vs head; auto protocol; parity
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -n 1 gpurun_out/pytest_gpu.log
G='{"scheds":["ag777","ag111","ring","ar822","ar56","ar_ring","a2a"],"sizes":[1024,4096,16384,65536,131072,262144,524288],"knobs":[{}]}'
for i in 1 2; do
SCCL_LIB=$PWD/build/ab/libsccl_exec_head.so timeout 600 python tools/tune.py "$G" > gpurun_out/llg_head_$i.jsonl 2>&1
timeout 600 python tools/tune.py "$G" > gpurun_out/llg_new_$i.jsonl 2>&1
done
