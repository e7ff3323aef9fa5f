python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python tools/tune.py '{"scheds":["null1","ag111","ag777","ar822"],"sizes":[16,1024,8192],"knobs":[{}]}' > gpurun_out/tune_floor.jsonl 2>&1
