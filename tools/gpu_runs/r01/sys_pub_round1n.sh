# counter-release mode under system-scope signalling (loopback proxy of multi-process mode)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for m in 0 1; do
SCCL_LOOPBACK_SYS=1 SCCL_SELFPUB=$m python tools/tune.py '{"scheds":["ag777","ring","ar56","ar_ring","ar822","ag111","a2a"],"sizes":[262144,1048576,4194304,16777216],"knobs":[{"protocol":"simple"}]}' > gpurun_out/tune_syspub$m.jsonl 2>&1
SCCL_LOOPBACK_SYS=1 SCCL_SELFPUB=$m python tools/probes/trace_hops.py 16384:1 262144:8 > gpurun_out/trace_syspub$m.jsonl 2>&1
done
