# discard only for wide streaming reductions: parity + sizes
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
timeout 600 python tools/tune.py '{"scheds":["ar822","ar56","ar_ring","ag777"],"sizes":[67108864,134217728],"knobs":[{}]}' > gpurun_out/tune_discard2.jsonl 2>&1
