#!/bin/bash
# robustness after the plan-policy changes: multi-process tests (balanced groups), long fuzz
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multiprocess.py -x -q > gpurun_out/pytest_mp.log 2>&1; tail -n 1 gpurun_out/pytest_mp.log
timeout 900 python tools/fuzz_stress.py 2000 21 > gpurun_out/fuzz_stress_21.json 2>&1; cut -c1-200 gpurun_out/fuzz_stress_21.json
