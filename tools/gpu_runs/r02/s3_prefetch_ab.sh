# round 2 session 3: producer prefetch of the next op's receipt counters, same-box A/B (SCCL_PREFETCH 0 vs 1) + trace
set -x
make -s -j8 all > /dev/null
timeout 900 python tools/probes/ab_env.py SCCL_PREFETCH 0 1 ar56:67108864 ar56:16777216 ar56:268435456 ar56f:67108864 ar_ring:67108864 ar_ring:16777216 ag777:134217728 ag777:16777216 ag_ring:16777216 ar822:67108864 a2a:67108864 ar56:1048576 ag777:1048576 > gpurun_out/s3_prefetch_ab.jsonl 2> gpurun_out/s3_prefetch_ab.err
for s in ar56 ar_ring; do timeout 300 python tools/probes/trace_chain.py $s 67108864; done > gpurun_out/s3_trace_chain3.jsonl 2>> gpurun_out/s3_prefetch_ab.err
cat gpurun_out/s3_prefetch_ab.jsonl
