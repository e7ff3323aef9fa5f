# round 2 session 3: multi-process fuzz, 500 cases per world (one rank per process, all on cuda:0, time-sliced): random schedules x modes, P = 2/3/4/8; plus the new GPU test
set -x
make -s -j8 all > /dev/null
for W in 2 3 4 8; do
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $W --master-addr 127.0.0.1 --master-port 2960$W tools/fuzz_multiproc.py 500 $((13 + W)) >> gpurun_out/s3_fuzz_mp500.jsonl 2>> gpurun_out/s3_fuzz_mp500.err
done
cat gpurun_out/s3_fuzz_mp500.jsonl
timeout 900 python -m pytest tests/test_gpu_multiprocess.py -k fuzz -x -q > gpurun_out/s3_fuzz_mp_test.log 2>&1; tail -1 gpurun_out/s3_fuzz_mp_test.log
