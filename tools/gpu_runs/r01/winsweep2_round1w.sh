#!/bin/bash
# window size x chunk groups again after the per-op overhead cuts
set -x
mkdir -p gpurun_out
python tools/tune.py '{"scheds":["ag777"],"sizes":[134217728],"knobs":[{},{"env":{"SCCL_WINDOW":32768}},{"env":{"SCCL_WINDOW":131072}},{"kc":1,"kb":37},{"kc":1,"kb":37,"env":{"SCCL_WINDOW":65536}},{"kc":1,"kb":37,"env":{"SCCL_WINDOW":131072}},{}]}' | tee gpurun_out/winsweep2.jsonl
python tools/tune.py '{"scheds":["ring","ar56","ar_ring"],"sizes":[134217728],"knobs":[{},{"env":{"SCCL_WINDOW":32768}},{"env":{"SCCL_WINDOW":65536}},{"env":{"SCCL_WINDOW":131072}},{"env":{"SCCL_WINDOW":262144}},{}]}' | tee -a gpurun_out/winsweep2.jsonl
