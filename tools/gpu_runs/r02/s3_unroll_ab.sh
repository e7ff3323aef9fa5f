# round 2 session 3: reduce loops with several vectors in flight per thread vs HEAD (streaming + mid sizes), parity
set -x
make -s -j8 all > /dev/null
W="ar56:67108864 ar56:16777216 ar56f:67108864 ar822:67108864 ar822f:67108864 ar_ring:67108864 ar_ringf:67108864 ar822:4194304 ar56:4194304 ag777:134217728"
for rep in 1 2 3; do
  SCCL_LIB=build/ab/libsccl_head.so timeout 600 python tools/probes/ab_env.py SCCL_NOP 0 1 $W | sed "s/^{/{\"lib\": \"head\", /" >> gpurun_out/s3_unroll_ab.jsonl
  timeout 600 python tools/probes/ab_env.py SCCL_NOP 0 1 $W | sed 's/^{/{"lib": "new", /' >> gpurun_out/s3_unroll_ab.jsonl
done 2> gpurun_out/s3_unroll_ab.err
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/s3_unroll_parity.log 2>&1; tail -1 gpurun_out/s3_unroll_parity.log
