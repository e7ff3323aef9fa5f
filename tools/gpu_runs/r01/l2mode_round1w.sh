#!/bin/bash
# relay receipts in L2: evict_last stores (1), plain stores (3), evict_last + demote after the forwarding load (5)
set -x
mkdir -p gpurun_out
python tools/tune.py '{"scheds":["ag777","ring","ar56","ar_ring","ar822"],"sizes":[134217728],"knobs":[{},{"env":{"SCCL_L2HINT":3}},{"env":{"SCCL_L2HINT":5}},{}]}' | tee gpurun_out/l2mode.jsonl
python tools/tune.py '{"scheds":["ag777"],"sizes":[67108864, 536870912],"knobs":[{},{"env":{"SCCL_L2HINT":3}},{"env":{"SCCL_L2HINT":5}}]}' | tee -a gpurun_out/l2mode.jsonl
