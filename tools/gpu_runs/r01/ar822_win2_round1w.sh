#!/bin/bash
mkdir -p gpurun_out
python tools/tune.py '{"scheds":["ar822"],"sizes":[16777216,67108864,134217728],"knobs":[{},{"env":{"SCCL_WINDOW":16384}},{"env":{"SCCL_WINDOW":8192}},{}]}' > gpurun_out/ar822_win2.jsonl 2>&1
python tools/tune.py '{"scheds":["ar56","ar_ring"],"sizes":[67108864,134217728],"knobs":[{},{"env":{"SCCL_WINDOW":16384}},{}]}' >> gpurun_out/ar822_win2.jsonl 2>&1
