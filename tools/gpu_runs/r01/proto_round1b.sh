# protocol crossover and stage knobs after the multi-storer change
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python tools/tune.py '{"scheds":["ag777","ag111","ring","ar822","ar56","ar_ring","a2a"],"sizes":[65536,131072,262144,524288,1048576,2097152,4194304,8388608,16777216],"knobs":[{"protocol":"ll"},{"protocol":"simple"}]}' > gpurun_out/tune_proto2.jsonl 2>&1
python tools/tune.py '{"scheds":["ag777","ag111","ar822","ar56","a2a"],"sizes":[4194304,67108864],"knobs":[{},{"budget":196608},{"tile":16384},{"tile":16384,"budget":49152},{"tile":65536,"budget":196608},{"tile":32768,"budget":196608}]}' > gpurun_out/tune_knobs2.jsonl 2>&1
