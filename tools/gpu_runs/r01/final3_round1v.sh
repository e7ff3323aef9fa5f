# round-1 evidence of the final kernel: parity, sweeps (cfg1-5), ncu captures, bench + reference arm
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
timeout 900 python tools/size_sweep.py > gpurun_out/size_sweep_v6.jsonl 2> gpurun_out/size_sweep_v6.err
timeout 900 python tools/pareto_sweep.py > gpurun_out/pareto_v6.jsonl 2> gpurun_out/pareto_v6.err
mkdir -p gpurun_out/prof6
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/prof6/launches.csv python bench.py --steps 3 --warmup 3 --no-sweep --cpu-seconds 0.2 --cpu-bytes 65536 > gpurun_out/prof6/ncu_launch_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:exec_kernel -s 4 -c 1 -o gpurun_out/prof6/ag777 python bench.py --steps 2 --warmup 3 --no-sweep --cpu-seconds 0.1 --cpu-bytes 65536 > gpurun_out/prof6/ncu_ag.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:exec_kernel -s 3 -c 1 -o gpurun_out/prof6/ar822 python tools/tune.py '{"scheds":["ar822"],"sizes":[67108864],"knobs":[{}]}' > gpurun_out/prof6/ncu_ar.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:exec_kernel -s 3 -c 1 -o gpurun_out/prof6/ar56 python tools/tune.py '{"scheds":["ar56"],"sizes":[67108864],"knobs":[{}]}' > gpurun_out/prof6/ncu_ar56.log 2>&1
timeout 400 python bench.py > gpurun_out/bench.log 2>&1
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.log 2>&1
