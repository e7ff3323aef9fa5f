#!/bin/bash
# protocol crossover sweep (loopback gpu scope and sys scope) after the per-op overhead cuts: refit predict_us
set -x
mkdir -p gpurun_out
G='{"scheds":["ag777","ag111","ring","ar822","ar56","ar_ring","a2a"],"sizes":[16384,65536,131072,262144,524288,1048576,2097152,4194304,8388608,16777216],"knobs":[{"protocol":"ll"},{"protocol":"simple"}]}'
timeout 900 python tools/tune.py "$G" > gpurun_out/proto_refit.jsonl 2>&1
SCCL_LOOPBACK_SYS=1 timeout 900 python tools/tune.py "$G" > gpurun_out/proto_refit_sys.jsonl 2>&1
python tools/fit_protocol.py gpurun_out/proto_refit.jsonl
python tools/fit_protocol.py gpurun_out/proto_refit_sys.jsonl
