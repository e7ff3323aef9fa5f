# AG (7,7,7) 128 MiB: smaller tiles / chunk groups under window-major + hints
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
SCCL_WINDOW=16384 timeout 600 python tools/tune.py '{"scheds":["ag777","ar56"],"sizes":[134217728],"knobs":[{"protocol":"simple","tile":16384},{"protocol":"simple","tile":16384,"budget":49152}]}' > gpurun_out/tune_win4.jsonl 2>&1
SCCL_WINDOW=32768 timeout 600 python tools/tune.py '{"scheds":["ag777"],"sizes":[134217728],"knobs":[{"protocol":"simple","kc":2,"kb":18},{"protocol":"simple","budget":196608},{"protocol":"simple","kb":36,"kc":1}]}' >> gpurun_out/tune_win4.jsonl 2>&1
SCCL_WINDOW=65536 timeout 600 python tools/tune.py '{"scheds":["ag777"],"sizes":[134217728],"knobs":[{"protocol":"simple","kc":2,"kb":18}]}' >> gpurun_out/tune_win4.jsonl 2>&1
