# storer warps publish their own counters in tile order (no signaler warp): parity, hop trace, sweep, bench
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
python tools/probes/trace_hops.py 16384:1 262144:8 1048576:32 > gpurun_out/trace_selfpub.jsonl 2>&1
python tools/tune.py '{"scheds":["ag777","ring","ar56","ar_ring","ar822","ag111","a2a"],"sizes":[262144,1048576,4194304,16777216,134217728],"knobs":[{"protocol":"simple"}]}' > gpurun_out/tune_selfpub.jsonl 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --no-sweep --cpu-seconds 1 > gpurun_out/bench.log 2>&1
