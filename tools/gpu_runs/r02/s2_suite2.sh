# round 2 session 2: GPU suite + fuzz after the simple-protocol chunk-group rule; bench latency sweep re-run
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/s2s_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -rs > gpurun_out/s2s_pytest_gpu.log 2>&1
timeout 900 python tools/fuzz_stress.py 400 > gpurun_out/s2s_fuzz.log 2>&1
timeout 900 python bench.py > gpurun_out/s2s_bench.log 2>&1
tail -3 gpurun_out/s2s_pytest_gpu.log; tail -3 gpurun_out/s2s_fuzz.log
