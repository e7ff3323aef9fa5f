#!/bin/bash
# LL relay/reduce chains: every chunk its own group (kc = G) with 1 or 2 byte parts
mkdir -p gpurun_out
python tools/tune.py '{"scheds":["ag777"],"sizes":[16384,65536,131072,262144,524288],"knobs":[{"protocol":"ll"},{"protocol":"ll","kc":56,"kb":1},{"protocol":"ll","kc":56,"kb":2}]}' > gpurun_out/llgrid2.jsonl 2>&1
python tools/tune.py '{"scheds":["ar56"],"sizes":[65536,262144,524288,1048576,2097152],"knobs":[{"protocol":"ll"},{"protocol":"ll","kc":56,"kb":1},{"protocol":"ll","kc":56,"kb":2}]}' >> gpurun_out/llgrid2.jsonl 2>&1
