# AR (8,2,2) stage configs now that its DRAM traffic is at the floor
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python tools/tune.py '{"scheds":["ar822"],"sizes":[67108864,268435456],"knobs":[{},{"tile":32768,"budget":98304},{"tile":49152,"budget":147456},{"tile":65536,"budget":131072},{"tile":40960,"budget":122880}]}' > gpurun_out/tune_ar822cfg.jsonl 2>&1
SCCL_WINDOW=131072 timeout 900 python tools/tune.py '{"scheds":["ar822"],"sizes":[67108864,268435456],"knobs":[{},{"tile":32768,"budget":98304}]}' >> gpurun_out/tune_ar822cfg.jsonl 2>&1
SCCL_WINDOW=262144 timeout 900 python tools/tune.py '{"scheds":["ar822"],"sizes":[67108864,268435456],"knobs":[{},{"tile":32768,"budget":98304}]}' >> gpurun_out/tune_ar822cfg.jsonl 2>&1
