#!/bin/bash
# do compute-warp discards remove the chain allreduces' scratch write-backs? DRAM bytes per launch
set -x
mkdir -p gpurun_out/ncu_l2
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct
for s in ar56 ar_ring; do
for d in 1; do
SCCL_DISCARD=$d SCCL_L2HINT=3 timeout 300 ncu --metrics $M --clock-control none -k regex:exec_kernel -s 3 -c 1 --csv --log-file gpurun_out/ncu_l2/${s}_d$d.csv python tools/tune.py "{\"scheds\":[\"$s\"],\"sizes\":[134217728],\"knobs\":[{}]}" > /dev/null 2>&1
done
SCCL_WINDOW=0 timeout 300 ncu --metrics $M --clock-control none -k regex:exec_kernel -s 3 -c 1 --csv --log-file gpurun_out/ncu_l2/${s}_w0.csv python tools/tune.py "{\"scheds\":[\"$s\"],\"sizes\":[134217728],\"knobs\":[{}]}" > /dev/null 2>&1
timeout 300 ncu --metrics $M --clock-control none -k regex:exec_kernel -s 3 -c 1 --csv --log-file gpurun_out/ncu_l2/${s}_16m.csv python tools/tune.py "{\"scheds\":[\"$s\"],\"sizes\":[16777216],\"knobs\":[{}]}" > /dev/null 2>&1
done
