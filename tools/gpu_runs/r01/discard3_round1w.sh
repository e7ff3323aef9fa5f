#!/bin/bash
# signaler discards (2) with relays stored plain (L2HINT=3) vs evict-last (1)
set -x
mkdir -p gpurun_out
python tools/tune.py '{"scheds":["ar56","ar_ring","ar822"],"sizes":[67108864,134217728],"knobs":[{},{"env":{"SCCL_DISCARD":2,"SCCL_L2HINT":3}},{"env":{"SCCL_DISCARD":1,"SCCL_L2HINT":3}},{"env":{"SCCL_DISCARD":2,"SCCL_L2HINT":1}},{}]}' | tee gpurun_out/discard3.jsonl
