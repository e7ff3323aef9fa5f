# windowed signaler (cross-op batches, ops prepared ahead) vs storer self-publish
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
SCCL_SELFPUB=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_gpu_selfpub.log 2>&1
for m in 0 1; do
SCCL_SELFPUB=$m python tools/probes/trace_hops.py 16384:1 262144:8 1048576:32 > gpurun_out/trace_win$m.jsonl 2>&1
SCCL_SELFPUB=$m python tools/tune.py '{"scheds":["ag777","ring","ar56","ar_ring","ar822","ag111","a2a"],"sizes":[65536,262144,1048576,4194304,16777216,134217728],"knobs":[{"protocol":"simple"}]}' > gpurun_out/tune_win$m.jsonl 2>&1
done
timeout 300 python bench.py --steps 20 --warmup 5 --no-sweep --cpu-seconds 1 > gpurun_out/bench.log 2>&1
