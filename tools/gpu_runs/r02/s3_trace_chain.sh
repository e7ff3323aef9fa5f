# round 2 session 3: per-CTA time breakdown (producer flag/empty waits, load, compute, store) of the streaming launches
set -x
make -s -j8 all > /dev/null
for s in ar56 ar_ring ar822; do timeout 300 python tools/probes/trace_chain.py $s 67108864; done > gpurun_out/s3_trace_chain.jsonl 2> gpurun_out/s3_trace_chain.err
timeout 300 python tools/probes/trace_chain.py ag777 134217728 >> gpurun_out/s3_trace_chain.jsonl 2>> gpurun_out/s3_trace_chain.err
cat gpurun_out/s3_trace_chain.jsonl; tail -5 gpurun_out/s3_trace_chain.err
