# round 2 session 3: epoch-parity LL slot sets (no entry handshake) -- new back-to-back test, then the GPU suite
set -x
make -s -j8 all > /dev/null
timeout 900 python -m pytest tests/test_gpu_ll_parity.py -x -q -rs > gpurun_out/s3_llparity.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -rs > gpurun_out/s3_pytest_gpu2.log 2>&1
tail -3 gpurun_out/s3_llparity.log; tail -3 gpurun_out/s3_pytest_gpu2.log
