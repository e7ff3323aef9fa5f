# multi-storer-warp kernel: parity, then the size sweep and the bench
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
timeout 900 python tools/size_sweep.py cfg2,cfg3,cfg4 > gpurun_out/size_sweep_v2.jsonl 2> gpurun_out/size_sweep_v2.err
timeout 300 python bench.py --steps 20 --warmup 5 --no-sweep --cpu-seconds 1 > gpurun_out/bench.log 2>&1
