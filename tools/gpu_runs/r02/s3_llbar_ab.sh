# round 2 session 3: LL kernel without the redundant end-of-op barrier vs HEAD; graph-timed LL sizes
set -x
make -s -j8 all > /dev/null
S="ag777:1024 ag777:65536 ag777:262144 ag111:1024 ag_ring:1024 ag_ring:65536 ag_ring:262144 ar56:1024 ar56:65536 ar56:1048576 ar_ring:1024 ar_ring:1048576 a2a:1024 a2a:65536 ar822:1024 ar822:65536"
for rep in 1 2 3; do
  SCCL_LIB=build/ab/libsccl_head.so AB_GRAPH=1 timeout 600 python tools/probes/ab_env.py SCCL_NOP 0 1 $S | sed "s/^{/{\"lib\": \"head\", /" >> gpurun_out/s3_llbar_ab.jsonl
  AB_GRAPH=1 timeout 600 python tools/probes/ab_env.py SCCL_NOP 0 1 $S | sed 's/^{/{"lib": "new", /' >> gpurun_out/s3_llbar_ab.jsonl
done 2> gpurun_out/s3_llbar_ab.err
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multiprocess.py tests/test_gpu_ll_parity.py tests/test_gpu_watchdog.py -x -q > gpurun_out/s3_llbar_parity.log 2>&1; tail -2 gpurun_out/s3_llocc_parity.log
