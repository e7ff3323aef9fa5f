#!/bin/bash
# LL one-shot allreduce: chunk groups vs byte parts (the 8-input reduce sits in one group)
mkdir -p gpurun_out
python tools/tune.py '{"scheds":["ar822"],"sizes":[16384,65536,262144],"knobs":[{"protocol":"ll"},{"protocol":"ll","kc":8,"kb":2},{"protocol":"ll","kc":8,"kb":4},{"protocol":"ll","kc":8,"kb":8},{"protocol":"ll","kc":4,"kb":4},{"protocol":"ll","kc":2,"kb":8},{"protocol":"ll","kc":1,"kb":16}]}' > gpurun_out/llsplit.jsonl 2>&1
python tools/tune.py '{"scheds":["ar56","ar_ring"],"sizes":[65536,262144,1048576],"knobs":[{"protocol":"ll"},{"protocol":"ll","kc":8,"kb":4},{"protocol":"ll","kc":16,"kb":2}]}' >> gpurun_out/llsplit.jsonl 2>&1
