# round 2 session 3: launch geometry by multiply-high instead of four divides in every CTA prologue vs HEAD; graph-timed LL sizes
set -x
make -s -j8 all > /dev/null
S="ag777:1024 ag777:65536 ag111:1024 ag111:4096 ag_ring:1024 ag_ring:65536 ar56:1024 ar56:65536 ar_ring:1024 a2a:1024 a2a:65536 ar822:1024 ar822:65536 ag111:65536 ag777:1048576"
for rep in 1 2 3; do
  SCCL_LIB=build/ab/libsccl_head.so AB_GRAPH=1 timeout 600 python tools/probes/ab_env.py SCCL_NOP 0 1 $S | sed "s/^{/{\"lib\": \"head\", /" >> gpurun_out/s3_fdiv_ab.jsonl
  AB_GRAPH=1 timeout 600 python tools/probes/ab_env.py SCCL_NOP 0 1 $S | sed 's/^{/{"lib": "new", /' >> gpurun_out/s3_fdiv_ab.jsonl
done 2> gpurun_out/s3_fdiv_ab.err
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multiprocess.py -x -q > gpurun_out/s3_fdiv_parity.log 2>&1; tail -2 gpurun_out/s3_llocc_parity.log
