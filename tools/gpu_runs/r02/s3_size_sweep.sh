# round 2 session 3: BASELINE configs 1-4 size sweep (1 KiB - 1 GiB per rank) with the final build; GPU suite with the new parity tests
set -x
make -s -j8 all > /dev/null
timeout 2400 python tools/size_sweep.py > gpurun_out/s3_size_sweep.jsonl 2> gpurun_out/s3_size_sweep.err
timeout 1500 python -m pytest tests -m gpu -x -q -rs > gpurun_out/s3h_pytest_gpu.log 2>&1
wc -l gpurun_out/s3_size_sweep.jsonl; tail -2 gpurun_out/s3h_pytest_gpu.log
