python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
python tools/tune.py '{"scheds":["ar822","ar56","ag777","ag111"],"sizes":[1048576,16777216,67108864],"knobs":[{}]}' > gpurun_out/tune_dyn.jsonl 2>&1
