#!/bin/bash
# FADD2 (add.rn.f32x2) in the multi-input f32 accumulation: special values, parity, same-box A/B
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -k special_values -q > gpurun_out/pytest_special_new.log 2>&1; tail -n 1 gpurun_out/pytest_special_new.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -n 1 gpurun_out/pytest_gpu.log
G='{"scheds":["ar822"],"sizes":[1048576,4194304,16777216,67108864,134217728],"knobs":[{}]}'
for i in 1 2; do
SCCL_LIB=$PWD/build/ab/libsccl_exec_head.so timeout 600 python tools/tune.py "$G" > gpurun_out/f2_head_$i.jsonl 2>&1
timeout 600 python tools/tune.py "$G" > gpurun_out/f2_new_$i.jsonl 2>&1
done
