# round 2 session 3: lazy wait checks, LL first-miss variants: v3 nanosleep(100) on the first miss, v4 sleep after 4 polls instead of 32
set -x
make -s -j8 all > /dev/null
S="ag777:65536 ag777:262144 ag111:65536 ar56:1048576 a2a:65536 a2a:262144 ag_ring:65536 ar822:65536 ag111:262144 ar822:262144"
for rep in 1 2 3; do
  SCCL_LIB=build/ab/libsccl_head.so AB_GRAPH=1 timeout 600 python tools/probes/ab_env.py SCCL_NOP 0 1 $S | sed "s/^{/{\"lib\": \"head\", /" >> gpurun_out/s3_lazy_ab3.jsonl
  AB_GRAPH=1 timeout 600 python tools/probes/ab_env.py SCCL_NOP 0 1 $S | sed 's/^{/{"lib": "new", /' >> gpurun_out/s3_lazy_ab3.jsonl
  SCCL_LIB=build/ab/libsccl_v3.so AB_GRAPH=1 timeout 600 python tools/probes/ab_env.py SCCL_NOP 0 1 $S | sed "s/^{/{\"lib\": \"v3\", /" >> gpurun_out/s3_lazy_ab3.jsonl
  SCCL_LIB=build/ab/libsccl_v4.so AB_GRAPH=1 timeout 600 python tools/probes/ab_env.py SCCL_NOP 0 1 $S | sed "s/^{/{\"lib\": \"v4\", /" >> gpurun_out/s3_lazy_ab3.jsonl
done 2> gpurun_out/s3_lazy_ab3.err
