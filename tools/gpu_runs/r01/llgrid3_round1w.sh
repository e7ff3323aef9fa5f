#!/bin/bash
# LL grids for 8-chunk schedules at 64-256 KiB: fewer, longer byte parts
mkdir -p gpurun_out
python tools/tune.py '{"scheds":["ring","ag111"],"sizes":[65536,131072,262144],"knobs":[{"protocol":"ll"},{"protocol":"ll","kc":8,"kb":8},{"protocol":"ll","kc":8,"kb":4},{"protocol":"ll","kc":4,"kb":8},{"protocol":"ll","kc":8,"kb":12}]}' > gpurun_out/llgrid3.jsonl 2>&1
python tools/tune.py '{"scheds":["ar_ring","ar822"],"sizes":[262144,524288],"knobs":[{"protocol":"ll"},{"protocol":"ll","kc":8,"kb":4},{"protocol":"ll","kc":8,"kb":8},{"protocol":"ll","kc":8,"kb":12}]}' >> gpurun_out/llgrid3.jsonl 2>&1
