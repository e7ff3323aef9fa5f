#!/bin/bash
# LL chains with >= 32 chunks of <= 40 KiB: one chunk per CTA (new) vs head; auto protocol; parity
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -n 1 gpurun_out/pytest_gpu.log
G='{"scheds":["ag777","ar56","a2a","ring","ar_ring"],"sizes":[16384,65536,131072,262144,524288,1048576,2097152],"knobs":[{},{"protocol":"ll"}]}'
for i in 1 2; do
SCCL_LIB=$PWD/build/ab/libsccl_exec_head.so timeout 600 python tools/tune.py "$G" > gpurun_out/llc_head_$i.jsonl 2>&1
timeout 600 python tools/tune.py "$G" > gpurun_out/llc_new_$i.jsonl 2>&1
done
