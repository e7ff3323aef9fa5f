python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python tools/tune.py '{"scheds":["ag777","ag111","ar822","ar56"],"sizes":[134217728],"knobs":[{},{"budget":98304},{"budget":98304,"tile":16384},{"tile":16384},{"budget":131072,"tile":65536}]}' > gpurun_out/tune1.jsonl 2>&1
python tools/tune.py '{"scheds":["ag777","ag111"],"sizes":[1048576,16777216],"knobs":[{},{"budget":98304},{"tile":8192},{"tile":16384,"budget":65536},{"kc":7},{"kc":7,"budget":98304}]}' > gpurun_out/tune2.jsonl 2>&1
python tools/tune.py '{"scheds":["ag777","ag111","ar822"],"sizes":[65536,262144],"knobs":[{"protocol":"ll"},{"protocol":"simple"},{"protocol":"simple","tile":4096}]}' > gpurun_out/tune3.jsonl 2>&1
