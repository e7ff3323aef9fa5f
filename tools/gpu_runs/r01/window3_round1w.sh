# window size with L2 hints on (128 MiB per rank)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for w in 32768 65536 131072 262144; do
SCCL_WINDOW=$w timeout 600 python tools/tune.py '{"scheds":["ag777","ar56"],"sizes":[134217728],"knobs":[{"protocol":"simple"},{"protocol":"simple","kc":7,"kb":5}]}' > gpurun_out/tune_win3_$w.jsonl 2>&1
SCCL_WINDOW=$w timeout 600 python tools/tune.py '{"scheds":["ring","ar_ring","ar822"],"sizes":[134217728],"knobs":[{"protocol":"simple"}]}' >> gpurun_out/tune_win3_$w.jsonl 2>&1
done
timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:exec_kernel -s 3 -c 1 --csv python tools/tune.py '{"scheds":["ring"],"sizes":[134217728],"knobs":[{}]}' > gpurun_out/ncu_ring.csv 2>&1
