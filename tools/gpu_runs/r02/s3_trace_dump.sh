# round 2 session 3: raw trace of (56,14,14) bf16 64 MiB, channels 0-1 of every rank
set -x
make -s -j8 all > /dev/null
TRACE_DUMP=gpurun_out/s3_trace_ar56.json timeout 300 python tools/probes/trace_chain.py ar56 67108864 > gpurun_out/s3_trace_dump.jsonl 2>&1
