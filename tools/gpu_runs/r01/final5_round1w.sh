# round-1 evidence after the packed 2-input bf16/f16 reduces: parity, sweeps, ncu, bench + reference arm, fuzz, sanitizer
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
timeout 900 python tools/size_sweep.py > gpurun_out/size_sweep_v8.jsonl 2> gpurun_out/size_sweep_v8.err
timeout 900 python tools/pareto_sweep.py > gpurun_out/pareto_v8.jsonl 2> gpurun_out/pareto_v8.err
mkdir -p gpurun_out/prof8
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/prof8/launches.csv python bench.py --steps 3 --warmup 3 --no-sweep --cpu-seconds 0.2 --cpu-bytes 65536 > gpurun_out/prof8/ncu_launch_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:exec_kernel -s 4 -c 1 -o gpurun_out/prof8/ag777 python bench.py --steps 2 --warmup 3 --no-sweep --cpu-seconds 0.1 --cpu-bytes 65536 > gpurun_out/prof8/ncu_ag.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:exec_kernel -s 3 -c 1 -o gpurun_out/prof8/ar822 python tools/tune.py '{"scheds":["ar822"],"sizes":[67108864],"knobs":[{}]}' > gpurun_out/prof8/ncu_ar.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:exec_kernel -s 3 -c 1 -o gpurun_out/prof8/ar56 python tools/tune.py '{"scheds":["ar56"],"sizes":[67108864],"knobs":[{}]}' > gpurun_out/prof8/ncu_ar56.log 2>&1
timeout 400 python bench.py > gpurun_out/bench.log 2>&1
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.log 2>&1
timeout 900 python tools/fuzz_stress.py 400 11 > gpurun_out/fuzz_stress_11.json 2> gpurun_out/fuzz_stress_11.err
rm -f gpurun_out/sanitize_summary.txt; timeout 1500 bash tools/gpu_sanitize.sh
