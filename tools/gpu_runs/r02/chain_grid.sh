# round 2: chain allreduce stage / CTA grid with receipt discards on
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python tools/tune.py '{"scheds":["ar56"],"sizes":[67108864],"knobs":[{},{"kb":18},{"kb":56},{"kb":74},{"tile":65536,"budget":196608},{"tile":65536,"budget":196608,"kb":18},{"tile":16384,"budget":98304},{"tile":16384,"budget":98304,"kb":74},{"tile":32768,"budget":196608},{"tile":49152,"budget":147456},{"env":{"SCCL_WINDOW":"65536"}},{"env":{"SCCL_WINDOW":"16384"}},{"env":{"SCCL_SELFPUB":"1"}}]}' > gpurun_out/r02e_chain_grid.jsonl 2>&1
timeout 600 python tools/tune.py '{"scheds":["ar_ring","ar56"],"sizes":[16777216,268435456],"knobs":[{},{"kb":18},{"tile":65536,"budget":196608}]}' >> gpurun_out/r02e_chain_grid.jsonl 2>&1
