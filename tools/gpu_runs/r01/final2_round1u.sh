# evidence for the window-major + L2-hint kernel, part 1: parity, sweeps, protocol refits
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
timeout 900 python tools/size_sweep.py > gpurun_out/size_sweep_v5.jsonl 2> gpurun_out/size_sweep_v5.err
timeout 900 python tools/pareto_sweep.py > gpurun_out/pareto_v5.jsonl 2> gpurun_out/pareto_v5.err
timeout 600 python tools/tune.py '{"scheds":["ag777","ag111","ring","ar822","ar56","ar_ring","a2a"],"sizes":[16384,65536,131072,262144,524288,1048576,2097152,4194304,8388608,16777216],"knobs":[{"protocol":"ll"},{"protocol":"simple"}]}' > gpurun_out/tune_proto5.jsonl 2>&1
SCCL_LOOPBACK_SYS=1 timeout 600 python tools/tune.py '{"scheds":["ag777","ag111","ring","ar822","ar56","ar_ring","a2a"],"sizes":[16384,65536,131072,262144,524288,1048576,2097152,4194304,8388608,16777216],"knobs":[{"protocol":"ll"},{"protocol":"simple"}]}' > gpurun_out/tune_proto5_sys.jsonl 2>&1
