# round 2 session 3: after the lazy-wait change -- GPU suite, fuzz, bench N=1 (latency table) and the reference arm
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/s3g_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -rs > gpurun_out/s3g_pytest_gpu.log 2>&1
timeout 900 python tools/fuzz_stress.py 400 > gpurun_out/s3g_fuzz.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/s3g_bench_ref.log 2>&1
timeout 900 python bench.py > gpurun_out/s3g_bench.log 2>&1
tail -2 gpurun_out/s3g_pytest_gpu.log; tail -1 gpurun_out/s3g_fuzz.log
