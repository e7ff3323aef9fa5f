# round 2: chain allreduces -- does dropping consumed RS receipts from L2 pay now (DRAM-bound at 1.49 GB)?
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python tools/tune.py '{"scheds":["ar56","ar_ring"],"sizes":[67108864,268435456],"knobs":[{},{"env":{"SCCL_DISCARD":"1"}},{"env":{"SCCL_DISCARD":"1","SCCL_L2HINT":"1"}},{"env":{"SCCL_L2HINT":"3"}},{"env":{"SCCL_DISCARD":"1","SCCL_L2HINT":"3"}}]}' > gpurun_out/r02d_chain_discard.jsonl 2>&1
SCCL_DISCARD=1 timeout 300 ncu --set full --clock-control none -k regex:exec_kernel -s 3 -c 1 -o gpurun_out/r02_prof_ar56_discard python tools/tune.py '{"scheds":["ar56"],"sizes":[67108864],"knobs":[{}]}' > gpurun_out/r02_ncu_ar56d.log 2>&1
