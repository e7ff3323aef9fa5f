#!/bin/bash
mkdir -p gpurun_out
python tools/tune.py '{"scheds":["ar822"],"sizes":[67108864,134217728],"knobs":[{},{"env":{"SCCL_WINDOW":65536}},{"env":{"SCCL_WINDOW":131072}},{"env":{"SCCL_WINDOW":0}},{"kc":2,"kb":18},{}]}' > gpurun_out/ar822_win.jsonl 2>&1
