# bench.py N>1 path with VMM (cuMem fd) region sharing, every rank on cuda:0
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for n in 2 4; do
SCCL_BENCH_SHARE_GPU=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29519 bench.py --gpus $n --steps 3 --warmup 3 --bytes 4194304 --mem vmm > gpurun_out/bench_multi_vmm_$n.log 2>&1
echo "n=$n rc=$?" >> gpurun_out/bench_multi_vmm_rc.txt
done
