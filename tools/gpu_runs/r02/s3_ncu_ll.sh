# round 2 session 3: ncu --set full with source counters of the LL kernel: AG (7,7,7) 64 KiB and AR (8,2,2) bf16 64 KiB (loopback)
set -x
make -s -j8 all > /dev/null
timeout 300 ncu --set full --clock-control none --import-source on -k regex:exec_ll_kernel -s 10 -c 1 -o gpurun_out/s3_prof_ll_ag777 python tools/tune.py '{"scheds":["ag777"],"sizes":[65536],"knobs":[{}]}' > gpurun_out/s3_ncu_ll1.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:exec_ll_kernel -s 10 -c 1 -o gpurun_out/s3_prof_ll_ar822 python tools/tune.py '{"scheds":["ar822"],"sizes":[65536],"knobs":[{}]}' > gpurun_out/s3_ncu_ll2.log 2>&1
ls -la gpurun_out/s3_prof_ll*
