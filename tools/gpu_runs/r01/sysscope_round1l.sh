# price of system-scope signalling (multi-process mode) measured in loopback: hop trace + sizes
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for sys in 0 1; do
SCCL_LOOPBACK_SYS=$sys python tools/probes/trace_hops.py 16384:1 262144:8 > gpurun_out/trace_sys$sys.jsonl 2>&1
SCCL_LOOPBACK_SYS=$sys python tools/tune.py '{"scheds":["ag777","ring","ar822","ag111"],"sizes":[1024,65536,1048576,16777216,134217728],"knobs":[{}]}' > gpurun_out/tune_sys$sys.jsonl 2>&1
done
