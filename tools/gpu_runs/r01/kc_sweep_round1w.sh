#!/bin/bash
# (7,7,7) allgather at 64/128 MiB: chunk groups x window size (relay re-reads from L2)
set -x
mkdir -p gpurun_out
mkdir -p gpurun_out
python tools/tune.py '{"scheds":["ag777"],"sizes":[67108864,134217728],"knobs":[{},
 {"env":{"SCCL_WINDOW":32768}},
 {"kc":4,"kb":9},{"kc":4,"kb":9,"env":{"SCCL_WINDOW":32768}},{"kc":4,"kb":9,"env":{"SCCL_WINDOW":65536}},
 {"kc":7,"kb":5},{"kc":7,"kb":5,"env":{"SCCL_WINDOW":32768}},{"kc":7,"kb":5,"env":{"SCCL_WINDOW":65536}},
 {"kc":7,"kb":5,"tile":16384,"env":{"SCCL_WINDOW":16384}},
 {"kc":7,"kb":6},{"kc":8,"kb":4},{}]}' | tee gpurun_out/kc_sweep.jsonl
python tools/tune.py '{"scheds":["ring"],"sizes":[134217728],"knobs":[{},{"env":{"SCCL_WINDOW":32768}},{"env":{"SCCL_WINDOW":65536}}]}' | tee -a gpurun_out/kc_sweep.jsonl
