#!/bin/bash
# one-shot allreduce: tile size x stage count
mkdir -p gpurun_out
python tools/tune.py '{"scheds":["ar822"],"sizes":[16777216,67108864,134217728],"knobs":[{},{"tile":16384},{"tile":65536,"budget":196608},{"tile":32768,"budget":196608},{"tile":16384,"budget":196608},{}]}' > gpurun_out/ar822_tiles.jsonl 2>&1
