# LL prologue: epoch, program range and first op loaded in parallel; outputs on their own warp; next op prefetched
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
for i in 1 2; do
SCCL_LIB=$PWD/build/ab/libsccl_exec_head.so timeout 600 python tools/tune.py '{"scheds":["null1","ag111","ag777","ring","ar822","ar56","ar_ring","a2a"],"sizes":[1024,16384,65536],"knobs":[{"protocol":"ll"}]}' > gpurun_out/tune_llpro_head_$i.jsonl 2>&1
timeout 600 python tools/tune.py '{"scheds":["null1","ag111","ag777","ring","ar822","ar56","ar_ring","a2a"],"sizes":[1024,16384,65536],"knobs":[{"protocol":"ll"}]}' > gpurun_out/tune_llpro_new_$i.jsonl 2>&1
done
python tools/probes/trace_ll.py > gpurun_out/trace_ll4.jsonl 2>&1
