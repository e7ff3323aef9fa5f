# round 2 session 3: ncu --set full with source counters of the chain allreduce (56,14,14) bf16 64 MiB (warp stall sampling per line)
set -x
make -s -j8 all > /dev/null
timeout 600 ncu --set full --clock-control none --import-source on -k regex:exec_kernel -s 3 -c 1 -o gpurun_out/s3_prof_ar56 python tools/tune.py '{"scheds":["ar56"],"sizes":[67108864],"knobs":[{}]}' > gpurun_out/s3_ncu_ar56.log 2>&1
ls -la gpurun_out/s3_prof_ar56.ncu-rep
