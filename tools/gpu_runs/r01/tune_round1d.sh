python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python tools/tune.py '{"scheds":["ar56"],"sizes":[67108864],"knobs":[{},{"tile":65536,"budget":196608},{"tile":49152,"budget":98304},{"tile":65536,"budget":131072},{"tile":16384,"budget":98304}]}' > gpurun_out/tune_ar56.jsonl 2>&1
python tools/tune.py '{"scheds":["ar822"],"sizes":[67108864],"knobs":[{},{"tile":98304,"budget":196608}]}' >> gpurun_out/tune_ar56.jsonl 2>&1
