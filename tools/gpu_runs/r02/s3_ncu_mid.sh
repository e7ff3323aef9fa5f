# round 2 session 3: ncu source sampling of the simple kernel at latency-bound mid sizes: AG (1,1,1) 256 KiB, AR (8,2,2) 1 MiB, AG (7,7,7) 1 MiB
set -x
make -s -j8 all > /dev/null
timeout 300 ncu --set full --clock-control none --import-source on -k regex:exec_kernel -s 10 -c 1 -o gpurun_out/s3_prof_mid_ag111 python tools/tune.py '{"scheds":["ag111"],"sizes":[262144],"knobs":[{}]}' > gpurun_out/s3_ncu_mid1.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:exec_kernel -s 10 -c 1 -o gpurun_out/s3_prof_mid_ar822 python tools/tune.py '{"scheds":["ar822"],"sizes":[1048576],"knobs":[{}]}' > gpurun_out/s3_ncu_mid2.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:exec_kernel -s 10 -c 1 -o gpurun_out/s3_prof_mid_ag777 python tools/tune.py '{"scheds":["ag777"],"sizes":[1048576],"knobs":[{}]}' > gpurun_out/s3_ncu_mid3.log 2>&1
ls gpurun_out/s3_prof_mid*
