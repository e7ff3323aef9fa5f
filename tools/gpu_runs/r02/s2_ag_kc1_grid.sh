# round 2 session 2: (7,7,7) allgather 128 MiB with one chunk group: window / tile / hint grid, 2 repeats
for rep in 1 2; do
timeout 900 python tools/tune.py '{"scheds":["ag777"],"sizes":[134217728],"knobs":[{},{"env":{"SCCL_WINDOW":"65536"}},{"env":{"SCCL_WINDOW":"16384"}},{"env":{"SCCL_WINDOW":"98304"}},{"tile":65536,"budget":196608},{"tile":16384,"budget":98304},{"tile":49152,"budget":147456},{"env":{"SCCL_L2HINT":"3"}},{"env":{"SCCL_L2HINT":"0"}},{"env":{"SCCL_WINDOW":"0"}},{"kb":36},{"kb":33},{"kb":30}]}' >> gpurun_out/s2_ag_kc1_grid.jsonl 2>&1
done
cat gpurun_out/s2_ag_kc1_grid.jsonl
