#!/bin/bash
# packed bf16/f16 add for 2-input reduces: special-value parity (head kernel and new) + same-box timing A/B
mkdir -p gpurun_out
SCCL_LIB=$PWD/build/ab/libsccl_exec_head.so timeout 600 python -m pytest tests/test_gpu_parity.py -k special_values -q > gpurun_out/pytest_special_head.log 2>&1; tail -1 gpurun_out/pytest_special_head.log
timeout 600 python -m pytest tests/test_gpu_parity.py -k special_values -q > gpurun_out/pytest_special_new.log 2>&1; tail -1 gpurun_out/pytest_special_new.log
G='{"scheds":["ar56","ar_ring","ar822"],"sizes":[1048576,16777216,67108864,134217728],"knobs":[{},{"protocol":"simple"}]}'
for i in 1 2; do
SCCL_LIB=$PWD/build/ab/libsccl_exec_head.so timeout 600 python tools/tune.py "$G" > gpurun_out/pair_head_$i.jsonl 2>&1
timeout 600 python tools/tune.py "$G" > gpurun_out/pair_new_$i.jsonl 2>&1
done
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
