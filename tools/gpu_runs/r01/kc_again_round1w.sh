#!/bin/bash
# (7,7,7) 128 MiB: chunk groups again after the per-op overhead cuts
mkdir -p gpurun_out
python tools/tune.py '{"scheds":["ag777"],"sizes":[134217728],"knobs":[{},{"kc":4,"kb":9},{"kc":4,"kb":9,"env":{"SCCL_WINDOW":65536}},{"kc":7,"kb":5},{"kc":7,"kb":5,"env":{"SCCL_WINDOW":65536}},{"kc":2,"kb":18,"env":{"SCCL_WINDOW":131072}},{}]}' > gpurun_out/kc_again.jsonl 2>&1
