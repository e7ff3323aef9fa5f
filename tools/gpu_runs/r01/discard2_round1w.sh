#!/bin/bash
# receipt discards by the signaler warp (2) vs compute warps (1) vs none (0), allreduce chains and one-shot
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -k window_major_forced -x -q > gpurun_out/pytest_discard2.log 2>&1; tail -2 gpurun_out/pytest_discard2.log
python tools/tune.py '{"scheds":["ar56","ar_ring","ar822"],"sizes":[67108864,134217728],"knobs":[{},{"env":{"SCCL_DISCARD":0}},{"env":{"SCCL_DISCARD":1}},{"env":{"SCCL_DISCARD":2}},{}]}' | tee gpurun_out/discard2.jsonl
