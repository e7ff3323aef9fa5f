# after the counter-release change: parity, protocol crossover sweep (refit), trace
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
python tools/tune.py '{"scheds":["ag777","ag111","ring","ar822","ar56","ar_ring","a2a"],"sizes":[16384,65536,131072,262144,524288,1048576,2097152,4194304,8388608,16777216],"knobs":[{"protocol":"ll"},{"protocol":"simple"}]}' > gpurun_out/tune_proto3.jsonl 2>&1
python tools/probes/trace_hops.py 16384:1 262144:8 1048576:32 > gpurun_out/trace_final.jsonl 2>&1
