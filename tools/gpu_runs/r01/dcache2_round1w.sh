#!/bin/bash
# descriptor cache: on from 4 ops (default) / from 1 op / off, same build, plus the pre-cache head build
set -x
mkdir -p gpurun_out
G='{"scheds":["ag777","ring","ar56","ar_ring","ar822","a2a"],"sizes":[262144,1048576,4194304,16777216,134217728],"knobs":[{},{"env":{"SCCL_DCACHE":0}},{"env":{"SCCL_DCACHE":1}}]}'
for i in 1 2; do
timeout 600 python tools/tune.py "$G" > gpurun_out/dcache2_new_$i.jsonl 2>&1
SCCL_LIB=$PWD/build/ab/libsccl_exec_head.so timeout 600 python tools/tune.py "$G" > gpurun_out/dcache2_head_$i.jsonl 2>&1
done
