# round 2 session 3: lazy wait checks, three builds: head / new (all lazy) / v2 (wait_ge keeps its first-miss abort check)
set -x
make -s -j8 all > /dev/null
S="ag777:65536 ag777:262144 ag111:65536 ar56:1048576 a2a:65536 a2a:262144 ag_ring:65536 ar822:65536 ag111:262144 ar822:262144"
for rep in 1 2 3; do
  SCCL_LIB=build/ab/libsccl_head.so AB_GRAPH=1 timeout 600 python tools/probes/ab_env.py SCCL_NOP 0 1 $S | sed "s/^{/{\"lib\": \"head\", /" >> gpurun_out/s3_lazy_ab2.jsonl
  AB_GRAPH=1 timeout 600 python tools/probes/ab_env.py SCCL_NOP 0 1 $S | sed 's/^{/{"lib": "new", /' >> gpurun_out/s3_lazy_ab2.jsonl
  SCCL_LIB=build/ab/libsccl_v2.so AB_GRAPH=1 timeout 600 python tools/probes/ab_env.py SCCL_NOP 0 1 $S | sed "s/^{/{\"lib\": \"v2\", /" >> gpurun_out/s3_lazy_ab2.jsonl
done 2> gpurun_out/s3_lazy_ab2.err
