#!/bin/bash
# evict_last hints vs the persisting-L2 set-aside (cudaLimitPersistingL2CacheSize)
set -x
mkdir -p gpurun_out
python tools/tune.py '{"scheds":["ag777","ring","ar56","ar822"],"sizes":[134217728],"knobs":[{},{"persist":33554432},{"persist":67108864},{"persist":100663296},{"persist":1073741824},{}]}' | tee gpurun_out/persist.jsonl
