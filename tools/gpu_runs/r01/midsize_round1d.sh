# mid-size channel partition knobs (chunk groups x byte parts) with the multi-storer kernel
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python tools/tune.py '{"scheds":["ag777","ar56","ar822","ring","ar_ring","a2a","ag111"],"sizes":[1048576,4194304,16777216],"knobs":[{"protocol":"simple"},{"protocol":"simple","kc":2,"kb":18},{"protocol":"simple","kc":4,"kb":9},{"protocol":"simple","kc":8,"kb":4},{"protocol":"simple","tile":16384},{"protocol":"simple","tile":8192}]}' > gpurun_out/tune_mid.jsonl 2>&1
