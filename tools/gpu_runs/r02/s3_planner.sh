# round 2 session 3: planner warp (waits receipt counters ahead of the producer): same-box A/B, trace, GPU suite
set -x
make -s -j8 all > /dev/null
timeout 900 python tools/probes/ab_env.py SCCL_PLANNER 0 1 ar56:67108864 ar56:16777216 ar56:268435456 ar56f:67108864 ar_ring:67108864 ar_ring:16777216 ag777:134217728 ag777:16777216 ag_ring:16777216 ar822:67108864 a2a:67108864 ar56:1048576 ag777:1048576 ar56:4194304 ag_ring:1048576 > gpurun_out/s3_planner_ab.jsonl 2> gpurun_out/s3_planner.err
timeout 300 python tools/probes/trace_chain.py ar56 67108864 > gpurun_out/s3_trace_planner.jsonl 2>> gpurun_out/s3_planner.err
cat gpurun_out/s3_planner_ab.jsonl
timeout 1500 python -m pytest tests -m gpu -x -q -rs > gpurun_out/s3_pytest_planner.log 2>&1
tail -3 gpurun_out/s3_pytest_planner.log
