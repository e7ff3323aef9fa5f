# round 2 session 2: re-verify the committed state (smoke, GPU suite, bench both arms)
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/s2_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -rs > gpurun_out/s2_pytest_gpu.log 2>&1
timeout 600 python bench.py --impl reference > gpurun_out/s2_bench_ref.log 2>&1
timeout 600 python bench.py > gpurun_out/s2_bench.log 2>&1
tail -3 gpurun_out/s2_pytest_gpu.log
tail -c 3000 gpurun_out/s2_bench.log
