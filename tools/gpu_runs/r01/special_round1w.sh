#!/bin/bash
# canonical-NaN oracles + packed 2-input bf16/f16 add: special-value parity, then the whole GPU suite
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -k special_values -q > gpurun_out/pytest_special_new.log 2>&1; tail -n 1 gpurun_out/pytest_special_new.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -n 1 gpurun_out/pytest_gpu.log
