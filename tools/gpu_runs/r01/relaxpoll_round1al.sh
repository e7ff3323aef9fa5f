# counter polls with relaxed loads + one acquire fence (A/B vs previous build)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
for i in 1 2; do
SCCL_LIB=$PWD/build/ab/libsccl_exec_head.so timeout 600 python tools/tune.py '{"scheds":["ag777","ring","ar822","ar56","ar_ring","a2a"],"sizes":[262144,1048576,4194304,16777216,134217728],"knobs":[{"protocol":"simple"}]}' > gpurun_out/tune_rp_head_$i.jsonl 2>&1
timeout 600 python tools/tune.py '{"scheds":["ag777","ring","ar822","ar56","ar_ring","a2a"],"sizes":[262144,1048576,4194304,16777216,134217728],"knobs":[{"protocol":"simple"}]}' > gpurun_out/tune_rp_new_$i.jsonl 2>&1
done
timeout 300 python tools/probes/trace_hops.py 16384:1 262144:8 > gpurun_out/trace_rp.jsonl 2>&1
