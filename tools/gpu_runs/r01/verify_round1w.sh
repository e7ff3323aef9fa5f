#!/bin/bash
# parity after a kernel/policy change + the policy's timing + a bench line
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
python tools/tune.py '{"scheds":["ag777","ring","ar56","ar_ring","ar822"],"sizes":[134217728],"knobs":[{}]}' | tee gpurun_out/verify_tune.jsonl
timeout 600 python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err; tail -c 3000 gpurun_out/bench.log
