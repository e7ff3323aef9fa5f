# protocol crossover with system-scope signalling (the multi-process mode's fences) in loopback
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
SCCL_LOOPBACK_SYS=1 python tools/tune.py '{"scheds":["ag777","ag111","ring","ar822","ar56","ar_ring","a2a"],"sizes":[16384,65536,131072,262144,524288,1048576,2097152,4194304,8388608,16777216],"knobs":[{"protocol":"ll"},{"protocol":"simple"}]}' > gpurun_out/tune_proto_sys.jsonl 2>&1
