#!/bin/bash
# same-box A/B: descriptor cache in shared memory (new) vs global descriptor loads (head)
set -x
mkdir -p gpurun_out
G='{"scheds":["ag777","ring","ar56","ar_ring","ar822","a2a"],"sizes":[65536,262144,1048576,4194304,16777216,134217728],"knobs":[{}]}'
for i in 1 2; do
SCCL_LIB=$PWD/build/ab/libsccl_exec_head.so timeout 600 python tools/tune.py "$G" > gpurun_out/dcache_head_$i.jsonl 2>&1
timeout 600 python tools/tune.py "$G" > gpurun_out/dcache_new_$i.jsonl 2>&1
done
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
