#!/bin/bash
# DRAM bytes per launch under the two relay policies (evict-last = L2HINT 1, default = 3)
set -x
mkdir -p gpurun_out/ncu_l2
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct
for h in 1 3; do
for s in ag777 ar56 ar_ring; do
SCCL_L2HINT=$h timeout 300 ncu --metrics $M --clock-control none -k regex:exec_kernel -s 3 -c 1 --csv --log-file gpurun_out/ncu_l2/${s}_h$h.csv python tools/tune.py "{\"scheds\":[\"$s\"],\"sizes\":[134217728],\"knobs\":[{}]}" > /dev/null 2>&1
done; done
