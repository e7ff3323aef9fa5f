# LL kernel with 4 slot loads in flight per thread: parity + LL timings
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k "ll or LL or protocol" > gpurun_out/pytest_ll.log 2>&1
python tools/tune.py '{"scheds":["ag777","ag111","ring","ar822","ar56","ar_ring","a2a"],"sizes":[1024,16384,65536,131072,262144,524288,1048576,2097152,4194304],"knobs":[{"protocol":"ll"}]}' > gpurun_out/tune_ll3.jsonl 2>&1
