# round 2 session 3: tools/tune.py --multi end to end with two processes on one GPU (path check of the NVLink refit; numbers are not NVLink), then load its table through SCCL_POLICY
set -x
make -s -j8 all > /dev/null
SCCL_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 tools/tune.py --multi '{"sizes":[4096,65536,1048576],"nchannels":[0,16],"out":"gpurun_out/s3_policy_multi_P2.json"}' > gpurun_out/s3_tune_multi.log 2>&1
cat gpurun_out/s3_policy_multi_P2.json
SCCL_POLICY=gpurun_out/s3_policy_multi_P2.json python -c "
import sys; sys.path.insert(0,'.')
from paper_2008_08708_b200 import sccl, schedules as S
p = sccl.Plan(S.to_json(S.one_shot_allgather(2)), 0, 2, 65536, sccl.U8, device=-1)
print('policy', p.info()['policy'])
" >> gpurun_out/s3_tune_multi.log 2>&1
tail -5 gpurun_out/s3_tune_multi.log
