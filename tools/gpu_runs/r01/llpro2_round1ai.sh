# LL prologue v2 (no uniform base-table read before the first op): A/B vs previous build
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k "ll or LL or protocol or rank_counts or multiprocess" > gpurun_out/pytest_ll2.log 2>&1
for i in 1 2; do
SCCL_LIB=$PWD/build/ab/libsccl_exec_head.so timeout 600 python tools/tune.py '{"scheds":["null1","ag111","ag777","ring","ar822","ar56","ar_ring","a2a"],"sizes":[1024,16384,65536],"knobs":[{"protocol":"ll"}]}' > gpurun_out/tune_llpro2_head_$i.jsonl 2>&1
timeout 600 python tools/tune.py '{"scheds":["null1","ag111","ag777","ring","ar822","ar56","ar_ring","a2a"],"sizes":[1024,16384,65536],"knobs":[{"protocol":"ll"}]}' > gpurun_out/tune_llpro2_new_$i.jsonl 2>&1
done
python tools/probes/trace_ll.py > gpurun_out/trace_ll5.jsonl 2>&1
