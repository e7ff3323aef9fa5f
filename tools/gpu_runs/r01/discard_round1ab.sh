# dead scratch receipts discarded from L2 (no write-back): parity, AR sizes, DRAM bytes
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
timeout 600 python tools/tune.py '{"scheds":["ar822","ar56","ar_ring","ag777","ring","a2a","ag111"],"sizes":[67108864,134217728,536870912],"knobs":[{}]}' > gpurun_out/tune_discard.jsonl 2>&1
timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:exec_kernel -s 3 -c 1 --csv python tools/tune.py '{"scheds":["ar822"],"sizes":[67108864],"knobs":[{}]}' > gpurun_out/ncu_disc_ar822.csv 2>&1
timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:exec_kernel -s 3 -c 1 --csv python tools/tune.py '{"scheds":["ar56"],"sizes":[67108864],"knobs":[{}]}' > gpurun_out/ncu_disc_ar56.csv 2>&1
