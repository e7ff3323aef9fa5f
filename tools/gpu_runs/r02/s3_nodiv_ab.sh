# round 2 session 3: no runtime divides on the tile path vs HEAD (two library builds, alternating processes)
set -x
make -s -j8 all > /dev/null
W="ar56:67108864 ar56:16777216 ar_ring:67108864 ag777:134217728 ag777:16777216 ar822:67108864 a2a:67108864 ar56:1048576 ag777:1048576 ag111:1048576"
for rep in 1 2 3; do
  SCCL_LIB=build/ab/libsccl_head.so timeout 600 python tools/probes/ab_env.py SCCL_NOP 0 1 $W | sed "s/^{/{\"lib\": \"head\", /" >> gpurun_out/s3_nodiv_ab.jsonl
  timeout 600 python tools/probes/ab_env.py SCCL_NOP 0 1 $W | sed 's/^{/{"lib": "new", /' >> gpurun_out/s3_nodiv_ab.jsonl
done 2> gpurun_out/s3_nodiv_ab.err
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/s3_nodiv_parity.log 2>&1; tail -2 gpurun_out/s3_nodiv_parity.log
