# round 2 session 2: (7,7,7) allgather at 64 MiB - 512 MiB per rank, current defaults and window / group variants
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 python tools/tune.py '{"scheds":["ag777"],"sizes":[67108864,100663296,134217728,201326592,268435456,536870912],"knobs":[{}]}' > gpurun_out/s2_ag_sizes.jsonl 2>&1
timeout 1500 python tools/tune.py '{"scheds":["ag777"],"sizes":[134217728],"knobs":[{"env":{"SCCL_WINDOW":"32768"}},{"env":{"SCCL_WINDOW":"131072"}},{"env":{"SCCL_WINDOW":"262144"}},{"kc":1,"kb":37},{"kc":3,"kb":12},{"kc":2,"kb":18,"env":{"SCCL_WINDOW":"131072"}}]}' >> gpurun_out/s2_ag_sizes.jsonl 2>&1
cat gpurun_out/s2_ag_sizes.jsonl
