# window-major execution (receipts re-read from L2): parity, sizes (window vs op-major), DRAM bytes, bench
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
for w in 0 32768 65536 131072; do
SCCL_WINDOW=$w timeout 600 python tools/tune.py '{"scheds":["ag777","ring","ar56","ar_ring","ar822","ag111","a2a"],"sizes":[1048576,4194304,16777216,134217728],"knobs":[{"protocol":"simple"}]}' > gpurun_out/tune_win_$w.jsonl 2>&1
done
timeout 400 python bench.py --no-sweep --cpu-seconds 1 > gpurun_out/bench.log 2>&1
timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:exec_kernel -s 4 -c 1 --csv python bench.py --steps 2 --warmup 3 --no-sweep --cpu-seconds 0.1 --cpu-bytes 65536 > gpurun_out/ncu_win_ag.csv 2>&1
