#!/bin/bash
# LL grid size: default (up to 148 CTAs per rank) vs capped channel counts
mkdir -p gpurun_out
python tools/tune.py '{"scheds":["ag777"],"sizes":[65536,131072,262144],"knobs":[{"protocol":"ll"},{"protocol":"ll","kc":28,"kb":2},{"protocol":"ll","kc":21,"kb":3},{"protocol":"ll","kc":14,"kb":4},{"protocol":"ll","kc":56,"kb":1},{"protocol":"ll","kc":28,"kb":4}]}' > gpurun_out/llgrid.jsonl 2>&1
python tools/tune.py '{"scheds":["ar56"],"sizes":[262144,1048576],"knobs":[{"protocol":"ll"},{"protocol":"ll","kc":28,"kb":2},{"protocol":"ll","kc":56,"kb":1},{"protocol":"ll","kc":14,"kb":4},{"protocol":"ll","kc":28,"kb":4}]}' >> gpurun_out/llgrid.jsonl 2>&1
python tools/tune.py '{"scheds":["a2a"],"sizes":[65536,131072,262144],"knobs":[{"protocol":"ll"},{"protocol":"ll","kc":32,"kb":2},{"protocol":"ll","kc":16,"kb":4},{"protocol":"ll","kc":64,"kb":1},{"protocol":"ll","kc":16,"kb":8}]}' >> gpurun_out/llgrid.jsonl 2>&1
