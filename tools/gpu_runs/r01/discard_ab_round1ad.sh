# A/B in one run: previous build (no discard code) vs current build (discard only for wide reductions)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for i in 1 2; do
SCCL_LIB=$PWD/build/ab/libsccl_exec_head.so timeout 600 python tools/tune.py '{"scheds":["ar822","ar56","ar_ring","ag777"],"sizes":[67108864,134217728],"knobs":[{}]}' > gpurun_out/tune_ab_head_$i.jsonl 2>&1
timeout 600 python tools/tune.py '{"scheds":["ar822","ar56","ar_ring","ag777"],"sizes":[67108864,134217728],"knobs":[{}]}' > gpurun_out/tune_ab_new_$i.jsonl 2>&1
done
