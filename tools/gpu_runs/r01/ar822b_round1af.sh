# streaming wide reductions at 2 CTAs/SM: parity + sizes
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
timeout 900 python tools/tune.py '{"scheds":["ar822"],"sizes":[16777216,67108864,268435456,1073741824],"knobs":[{}]}' > gpurun_out/tune_ar822b.jsonl 2>&1
