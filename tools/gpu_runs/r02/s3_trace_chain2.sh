# round 2 session 3: receipt waits by program position (chain allreduces)
set -x
make -s -j8 all > /dev/null
for s in ar56 ar_ring; do timeout 300 python tools/probes/trace_chain.py $s 67108864; done > gpurun_out/s3_trace_chain2.jsonl 2> gpurun_out/s3_trace_chain2.err
