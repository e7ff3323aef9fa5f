#!/bin/bash
mkdir -p gpurun_out
python tools/tune.py '{"scheds":["ring","ag111"],"sizes":[262144,524288],"knobs":[{"protocol":"ll"},{"protocol":"ll","kc":2,"kb":55},{"protocol":"ll","kc":3,"kb":37},{"protocol":"ll","kc":4,"kb":27},{"protocol":"ll","kc":8,"kb":13}]}' > gpurun_out/llgrid4.jsonl 2>&1
