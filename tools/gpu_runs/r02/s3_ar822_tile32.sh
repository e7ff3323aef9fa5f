# round 2 session 3: pulled one-shot allreduce, 32 KiB tiles up to 512 KiB chunks (was 16 KiB) vs HEAD; parity
set -x
make -s -j8 all > /dev/null
W="ar822:524288 ar822:1048576 ar822:2097152 ar822:4194304 ar822:8388608 ar822f:1048576 ar822f:4194304 ar822:16777216"
for rep in 1 2 3; do
  SCCL_LIB=build/ab/libsccl_head.so AB_GRAPH=1 timeout 600 python tools/probes/ab_env.py SCCL_NOP 0 1 $W | sed "s/^{/{\"lib\": \"head\", /" >> gpurun_out/s3_ar822_tile32.jsonl
  AB_GRAPH=1 timeout 600 python tools/probes/ab_env.py SCCL_NOP 0 1 $W | sed 's/^{/{"lib": "new", /' >> gpurun_out/s3_ar822_tile32.jsonl
done 2> gpurun_out/s3_ar822_tile32.err
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/s3_ar822_tile32_parity.log 2>&1; tail -1 gpurun_out/s3_ar822_tile32_parity.log
