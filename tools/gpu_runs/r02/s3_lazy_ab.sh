# round 2 session 3: waits read the abort word / clock only after 1024 polls (not on the first miss): A/B vs HEAD, graph-timed small sizes + streaming sizes
set -x
make -s -j8 all > /dev/null
S="ag777:1024 ag777:65536 ag777:262144 ag777:1048576 ag111:1024 ag111:65536 ar822:1024 ar822:65536 ar822:1048576 ar56:65536 ar56:1048576 a2a:8192 a2a:65536 ag_ring:65536 ar_ring:65536"
L="ag777:134217728 ar56:67108864 ar822:67108864 ar_ring:16777216"
for rep in 1 2 3; do
  SCCL_LIB=build/ab/libsccl_head.so AB_GRAPH=1 timeout 600 python tools/probes/ab_env.py SCCL_NOP 0 1 $S | sed "s/^{/{\"lib\": \"head\", /" >> gpurun_out/s3_lazy_ab.jsonl
  AB_GRAPH=1 timeout 600 python tools/probes/ab_env.py SCCL_NOP 0 1 $S | sed 's/^{/{"lib": "new", /' >> gpurun_out/s3_lazy_ab.jsonl
done 2> gpurun_out/s3_lazy_ab.err
for rep in 1 2; do
  SCCL_LIB=build/ab/libsccl_head.so timeout 600 python tools/probes/ab_env.py SCCL_NOP 0 1 $L | sed "s/^{/{\"lib\": \"head\", /" >> gpurun_out/s3_lazy_ab.jsonl
  timeout 600 python tools/probes/ab_env.py SCCL_NOP 0 1 $L | sed 's/^{/{"lib": "new", /' >> gpurun_out/s3_lazy_ab.jsonl
done 2>> gpurun_out/s3_lazy_ab.err
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_watchdog.py -x -q > gpurun_out/s3_lazy_parity.log 2>&1; tail -2 gpurun_out/s3_lazy_parity.log
