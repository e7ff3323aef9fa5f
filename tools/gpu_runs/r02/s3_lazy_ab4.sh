# round 2 session 3: lazy wait checks, LL first-miss variants: v5 sleep after 256 (LL) / 512 (counters) polls, v6 after 4096
set -x
make -s -j8 all > /dev/null
S="ag777:65536 ag777:262144 ag777:1048576 ag111:65536 ar56:65536 ar56:1048576 a2a:65536 a2a:8192 ag_ring:65536 ar_ring:65536 ar822:65536 ar822:1048576 ag111:1024 ar56:16777216"
for rep in 1 2 3; do
  SCCL_LIB=build/ab/libsccl_head.so AB_GRAPH=1 timeout 600 python tools/probes/ab_env.py SCCL_NOP 0 1 $S | sed "s/^{/{\"lib\": \"head\", /" >> gpurun_out/s3_lazy_ab4.jsonl
  AB_GRAPH=1 timeout 600 python tools/probes/ab_env.py SCCL_NOP 0 1 $S | sed 's/^{/{"lib": "new", /' >> gpurun_out/s3_lazy_ab4.jsonl
  SCCL_LIB=build/ab/libsccl_v5.so AB_GRAPH=1 timeout 600 python tools/probes/ab_env.py SCCL_NOP 0 1 $S | sed "s/^{/{\"lib\": \"v5\", /" >> gpurun_out/s3_lazy_ab4.jsonl
  SCCL_LIB=build/ab/libsccl_v6.so AB_GRAPH=1 timeout 600 python tools/probes/ab_env.py SCCL_NOP 0 1 $S | sed "s/^{/{\"lib\": \"v6\", /" >> gpurun_out/s3_lazy_ab4.jsonl
done 2> gpurun_out/s3_lazy_ab4.err
