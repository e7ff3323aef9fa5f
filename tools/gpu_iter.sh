# one GPU iteration: smoke, gpu tests, bench (+ optional ncu capture)
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1
if [ -n "$NCU" ]; then
timeout 400 ncu --set full --clock-control none --import-source on -k regex:exec_kernel -s 5 -c 1 -o gpurun_out/prof_$NCU python bench.py --steps 2 --warmup 5 --no-sweep --cpu-seconds 0.1 --cpu-bytes 65536 > gpurun_out/ncu_full.log 2>&1
fi
