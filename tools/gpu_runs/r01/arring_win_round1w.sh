#!/bin/bash
# ring allreduce: window size at 64 / 128 / 512 MiB
set -x
mkdir -p gpurun_out
python tools/tune.py '{"scheds":["ar_ring"],"sizes":[67108864,134217728,536870912],"knobs":[{},{"env":{"SCCL_WINDOW":262144}},{"env":{"SCCL_WINDOW":524288}},{"env":{"SCCL_WINDOW":0}},{}]}' | tee gpurun_out/arring_win.jsonl
python tools/tune.py '{"scheds":["ring"],"sizes":[67108864,536870912],"knobs":[{},{"env":{"SCCL_WINDOW":262144}},{}]}' | tee -a gpurun_out/arring_win.jsonl
