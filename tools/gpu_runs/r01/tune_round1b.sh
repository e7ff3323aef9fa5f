python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python tools/tune.py '{"scheds":["ag777","ag111","ar822","ar56"],"sizes":[4096,16384,65536,262144,1048576,4194304],"knobs":[{"protocol":"ll"},{"protocol":"simple"}]}' > gpurun_out/tune_proto.jsonl 2>&1
