# LL copy path with 4 pairs in flight per thread (64 regs, 4 CTAs/SM): parity + LL sweep
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
timeout 600 python tools/tune.py '{"scheds":["ag777","ag111","ring","ar822","ar56","ar_ring","a2a"],"sizes":[1024,16384,65536,131072,262144,524288,1048576,2097152,4194304],"knobs":[{"protocol":"ll"}]}' > gpurun_out/tune_llcopy.jsonl 2>&1
