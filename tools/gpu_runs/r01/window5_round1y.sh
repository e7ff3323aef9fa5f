# AG (7,7,7) / AR (56,14,14) 128 MiB: chunk groups x window under window-major + hints
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for w in 65536 98304 131072; do
SCCL_WINDOW=$w timeout 600 python tools/tune.py '{"scheds":["ag777","ar56"],"sizes":[134217728],"knobs":[{"protocol":"simple","kc":2,"kb":18},{"protocol":"simple","kc":4,"kb":9},{"protocol":"simple","kc":3,"kb":12}]}' >> gpurun_out/tune_win5.jsonl 2>&1
done
