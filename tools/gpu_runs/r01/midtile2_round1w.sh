#!/bin/bash
# mid sizes, simple protocol: default tile vs 16 KiB / 32 KiB tiles (more CTAs when chunks are small)
mkdir -p gpurun_out
python tools/tune.py '{"scheds":["ar822","ar_ring","ar56","ag777","ring","ag111","a2a"],"sizes":[262144,524288,1048576,2097152,4194304,8388608,16777216],"knobs":[{"protocol":"simple"},{"protocol":"simple","tile":16384},{"protocol":"simple","tile":32768}]}' > gpurun_out/midtile2.jsonl 2>&1
