# round 2 session 2: chain allreduces at 64 MiB/rank over chunk groups x byte parts x windows
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 python tools/tune.py '{"scheds":["ar56"],"sizes":[67108864],"knobs":[{},{"kc":2,"kb":18},{"kc":4,"kb":9},{"kc":7,"kb":5},{"kc":8,"kb":4},{"kc":14,"kb":2},{"kc":28,"kb":1},{"kc":7,"kb":5,"env":{"SCCL_WINDOW":"65536"}},{"kc":7,"kb":5,"env":{"SCCL_WINDOW":"262144"}},{"kc":7,"kb":5,"env":{"SCCL_WINDOW":"0"}},{"kc":8,"kb":4,"env":{"SCCL_WINDOW":"65536"}},{"kc":14,"kb":2,"env":{"SCCL_WINDOW":"65536"}},{"kc":7,"kb":2},{"kc":7,"kb":3},{"kc":7,"kb":5,"tile":16384,"budget":98304}]}' > gpurun_out/s2_chain_groups.jsonl 2>&1
timeout 900 python tools/tune.py '{"scheds":["ar_ring"],"sizes":[67108864],"knobs":[{},{"kc":2,"kb":18},{"kc":4,"kb":9},{"kc":8,"kb":4}]}' >> gpurun_out/s2_chain_groups.jsonl 2>&1
cat gpurun_out/s2_chain_groups.jsonl
