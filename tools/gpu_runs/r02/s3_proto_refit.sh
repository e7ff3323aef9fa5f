# round 2 session 3: protocol crossover sweep (gpu and sys scope) with the final session-3 kernels; regret of the current constants and a refit
set -x
make -s -j8 all > /dev/null
G='{"scheds":["ag777","ag111","ring","ar822","ar56","ar_ring","a2a"],"sizes":[16384,32768,65536,131072,262144,524288,1048576,2097152,4194304,8388608,16777216],"knobs":[{"protocol":"ll"},{"protocol":"simple"}]}'
timeout 900 python tools/tune.py "$G" > gpurun_out/s3_proto.jsonl 2>&1
SCCL_LOOPBACK_SYS=1 timeout 900 python tools/tune.py "$G" > gpurun_out/s3_proto_sys.jsonl 2>&1
python tools/fit_protocol.py gpurun_out/s3_proto.jsonl --eval 4.80,0.522,0.353,4.50,2.72,0.126
python tools/fit_protocol.py gpurun_out/s3_proto_sys.jsonl --eval 4.79,0.520,0.353,5.00,6.33,0.163
