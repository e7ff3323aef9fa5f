#!/bin/bash
# storer warps keep one tile's writes in flight past its stage (signaler mode): parity, fuzz, same-box A/B
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -n 1 gpurun_out/pytest_gpu.log
timeout 600 python tools/fuzz_stress.py 300 10 > gpurun_out/fuzz_defer.json 2>&1; cut -c1-200 gpurun_out/fuzz_defer.json
G='{"scheds":["ag777","ring","ag111","a2a","ar56","ar_ring","ar822"],"sizes":[4194304,16777216,67108864,134217728],"knobs":[{}]}'
for i in 1 2; do
SCCL_LIB=$PWD/build/ab/libsccl_exec_head.so timeout 600 python tools/tune.py "$G" > gpurun_out/defer_head_$i.jsonl 2>&1
timeout 600 python tools/tune.py "$G" > gpurun_out/defer_new_$i.jsonl 2>&1
done
