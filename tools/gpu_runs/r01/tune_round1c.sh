python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python tools/tune.py '{"scheds":["ar56"],"sizes":[67108864],"knobs":[{},{"kc":7,"kb":5},{"kc":4,"kb":9},{"kc":2,"kb":18},{"kc":8,"kb":4},{"kc":14,"kb":2}]}' > gpurun_out/tune_kc.jsonl 2>&1
python tools/tune.py '{"scheds":["ag777"],"sizes":[16777216,134217728],"knobs":[{},{"kc":7,"kb":5},{"kc":2,"kb":18}]}' >> gpurun_out/tune_kc.jsonl 2>&1
python tools/tune.py '{"scheds":["ar822"],"sizes":[67108864],"knobs":[{},{"tile":32768,"budget":196608},{"tile":49152,"budget":196608},{"tile":65536,"budget":196608},{"tile":32768,"budget":98304},{"tile":65536,"budget":131072}]}' >> gpurun_out/tune_kc.jsonl 2>&1
