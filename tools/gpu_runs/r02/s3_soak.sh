# round 2 session 3: soak -- 2000-case random-schedule fuzz, the GPU suite twice, eight-process harness with bursts
set -x
make -s -j8 all > /dev/null
timeout 1800 python tools/fuzz_stress.py 2000 > gpurun_out/s3_soak_fuzz2000.log 2>&1
for i in 1 2; do timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s3_soak_suite$i.log 2>&1; done
SCCL_MULTIDEVICE_SHARE=1 SCCL_MULTIDEVICE_WORLD=4 timeout 1500 python -m pytest tests/test_gpu_multidevice.py -x -q -k one_rank > gpurun_out/s3_soak_multidev4.log 2>&1
tail -1 gpurun_out/s3_soak_fuzz2000.log; tail -1 gpurun_out/s3_soak_suite1.log; tail -1 gpurun_out/s3_soak_suite2.log; tail -1 gpurun_out/s3_soak_multidev4.log
