# round 2: new bench.py (per-rank value, full e2e, reference arm from schedule files), shared-GPU
# multi-process bench, ncu of the pull allreduce and the alltoall
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/r02c_bench_ref.log 2>&1
timeout 900 python bench.py > gpurun_out/r02c_bench.log 2>&1
SCCL_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --bytes 16777216 > gpurun_out/r02c_bench_share2.log 2>&1
SCCL_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 8 --steps 3 --warmup 3 --bytes 4194304 > gpurun_out/r02c_bench_share8.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:exec_kernel -s 3 -c 1 -o gpurun_out/r02_prof_ar822pull python tools/tune.py '{"scheds":["ar822"],"sizes":[67108864],"knobs":[{}]}' > gpurun_out/r02_ncu_ar822.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:exec_kernel -s 3 -c 1 -o gpurun_out/r02_prof_ar56 python tools/tune.py '{"scheds":["ar56"],"sizes":[67108864],"knobs":[{}]}' > gpurun_out/r02_ncu_ar56.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:exec_kernel -s 3 -c 1 -o gpurun_out/r02_prof_a2a python tools/tune.py '{"scheds":["a2a"],"sizes":[67108864],"knobs":[{}]}' > gpurun_out/r02_ncu_a2a.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/r02_launches_bench.csv python bench.py --steps 3 --warmup 3 --no-sweep --cpu-seconds 0.2 --cpu-bytes 65536 > gpurun_out/r02_ncu_launch_bench.log 2>&1
