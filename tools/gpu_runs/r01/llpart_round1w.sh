#!/bin/bash
# LL byte-part size (bytes of a chunk one CTA owns): 4096 (current) vs 2048 vs 1024
mkdir -p gpurun_out
G='{"scheds":["ag777","ag111","ring","ar822","ar56","ar_ring","a2a"],"sizes":[1024,4096,16384,65536,131072,262144,524288],"knobs":[{"protocol":"ll"},{"protocol":"ll","env":{"SCCL_LL_PART":2048}},{"protocol":"ll","env":{"SCCL_LL_PART":1024}}]}'
python tools/tune.py "$G" > gpurun_out/llpart_1.jsonl 2>&1
python tools/tune.py "$G" > gpurun_out/llpart_2.jsonl 2>&1
