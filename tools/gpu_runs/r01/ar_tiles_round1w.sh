#!/bin/bash
# allreduce chains: tile size x stage count (in-flight tiles per CTA)
set -x
mkdir -p gpurun_out
python tools/tune.py '{"scheds":["ar56","ar_ring"],"sizes":[16777216,134217728],"knobs":[{},{"tile":16384},{"tile":16384,"budget":196608},{"tile":65536,"budget":196608},{"tile":32768,"budget":196608},{}]}' | tee gpurun_out/ar_tiles.jsonl
