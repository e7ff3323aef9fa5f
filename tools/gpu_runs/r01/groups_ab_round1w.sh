#!/bin/bash
# balanced chunk-group assignment (new) vs chunk % kc (head): parity, fuzz, same-box A/B
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -n 1 gpurun_out/pytest_gpu.log
timeout 600 python tools/fuzz_stress.py 300 13 > gpurun_out/fuzz_groups.json 2>&1; cut -c1-120 gpurun_out/fuzz_groups.json
G='{"scheds":["a2a","ag777","ring","ag111","ar56","ar_ring","ar822"],"sizes":[65536,262144,1048576,4194304,16777216,134217728],"knobs":[{}]}'
for i in 1 2; do
SCCL_LIB=$PWD/build/ab/libsccl_exec_head.so timeout 600 python tools/tune.py "$G" > gpurun_out/grp_head_$i.jsonl 2>&1
timeout 600 python tools/tune.py "$G" > gpurun_out/grp_new_$i.jsonl 2>&1
done
