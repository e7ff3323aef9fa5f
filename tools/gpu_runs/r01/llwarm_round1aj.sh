# LL: constant-cache warm-up of the base table during the prologue (A/B vs previous build)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k "ll or LL or protocol or rank_counts" > gpurun_out/pytest_llw.log 2>&1
for i in 1 2 3; do
SCCL_LIB=$PWD/build/ab/libsccl_exec_head.so timeout 600 python tools/tune.py '{"scheds":["null1","ag111","ag777","ring","ar822","ar56","ar_ring","a2a"],"sizes":[1024,16384,65536],"knobs":[{"protocol":"ll"}]}' > gpurun_out/tune_llw_head_$i.jsonl 2>&1
timeout 600 python tools/tune.py '{"scheds":["null1","ag111","ag777","ring","ar822","ar56","ar_ring","a2a"],"sizes":[1024,16384,65536],"knobs":[{"protocol":"ll"}]}' > gpurun_out/tune_llw_new_$i.jsonl 2>&1
done
