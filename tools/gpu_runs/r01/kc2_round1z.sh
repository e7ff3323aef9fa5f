# AG (7,7,7): two chunk groups for streaming relay schedules
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
timeout 600 python tools/tune.py '{"scheds":["ag777"],"sizes":[16777216,67108864,134217728,536870912],"knobs":[{}]}' > gpurun_out/tune_kc2.jsonl 2>&1
SCCL_WINDOW=32768 timeout 600 python tools/tune.py '{"scheds":["ag777"],"sizes":[16777216,67108864,134217728,536870912],"knobs":[{"kc":1,"kb":37}]}' >> gpurun_out/tune_kc2.jsonl 2>&1
timeout 400 python bench.py --no-sweep --cpu-seconds 1 > gpurun_out/bench.log 2>&1
timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:exec_kernel -s 4 -c 1 --csv python bench.py --steps 2 --warmup 3 --no-sweep --cpu-seconds 0.1 --cpu-bytes 65536 > gpurun_out/ncu_kc2.csv 2>&1
