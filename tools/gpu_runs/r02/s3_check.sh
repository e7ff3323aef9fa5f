# round 2 session 3: state check after the container re-creation (smoke, GPU suite, bench N=1, reference arm)
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/s3_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -rs > gpurun_out/s3_pytest_gpu.log 2>&1
timeout 900 python bench.py > gpurun_out/s3_bench.log 2>&1
timeout 600 python bench.py --impl reference > gpurun_out/s3_bench_ref.log 2>&1
tail -3 gpurun_out/s3_pytest_gpu.log; tail -c 600 gpurun_out/s3_bench.log
