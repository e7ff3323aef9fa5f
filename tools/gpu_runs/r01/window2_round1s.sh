# window-major: chunk groups x window size at 128 MiB (L2 reuse of relayed receipts)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for w in 32768 65536 131072 262144; do
SCCL_WINDOW=$w timeout 600 python tools/tune.py '{"scheds":["ag777","ar56"],"sizes":[134217728],"knobs":[{"protocol":"simple"},{"protocol":"simple","kc":7,"kb":5},{"protocol":"simple","kc":2,"kb":18}]}' > gpurun_out/tune_win2_$w.jsonl 2>&1
SCCL_WINDOW=$w timeout 600 python tools/tune.py '{"scheds":["ring","ar_ring","ar822"],"sizes":[134217728],"knobs":[{"protocol":"simple"}]}' >> gpurun_out/tune_win2_$w.jsonl 2>&1
done
