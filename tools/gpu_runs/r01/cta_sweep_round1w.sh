#!/bin/bash
# (7,7,7) allgather at 64/128 MiB: fewer CTAs (shorter relay distance in L2) x stage depth
set -x
mkdir -p gpurun_out
python tools/tune.py '{"scheds":["ag777"],"sizes":[67108864,134217728],"knobs":[{},
 {"kc":2,"kb":9},{"kc":2,"kb":9,"budget":196608},{"kc":2,"kb":9,"tile":65536,"budget":196608},
 {"kc":1,"kb":18},{"kc":1,"kb":18,"budget":196608},{"kc":1,"kb":18,"tile":65536,"budget":196608},
 {"kc":2,"kb":12},{"kc":2,"kb":14},{"kc":2,"kb":16},
 {"kc":2,"kb":9,"budget":196608,"env":{"SCCL_WINDOW":32768}},{"kc":2,"kb":9,"budget":196608,"env":{"SCCL_WINDOW":131072}},{}]}' | tee gpurun_out/cta_sweep.jsonl
python tools/tune.py '{"scheds":["ring"],"sizes":[134217728],"knobs":[{},{"kc":1,"kb":18,"budget":196608},{"kc":1,"kb":18,"tile":65536,"budget":196608}]}' | tee -a gpurun_out/cta_sweep.jsonl
