#!/bin/bash
# L2 hint variants: 1 current; 3 relays plain; 11 relays+final stores plain; 19 relays plain + loads plain; 27 all plain (windowed)
set -x
mkdir -p gpurun_out
python tools/tune.py '{"scheds":["ag777","ring","ar56","ar_ring","ar822","a2a"],"sizes":[134217728],"knobs":[{},{"env":{"SCCL_L2HINT":3}},{"env":{"SCCL_L2HINT":11}},{"env":{"SCCL_L2HINT":19}},{"env":{"SCCL_L2HINT":27}},{"env":{"SCCL_L2HINT":0}},{}]}' | tee gpurun_out/l2mode2.jsonl
