# LL kernel reads its packed program in one load (offsets in kernel params): parity, trace, small-size latency
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
python tools/probes/trace_ll.py > gpurun_out/trace_ll2.jsonl 2>&1
python tools/tune.py '{"scheds":["null1","ag111","ag777","ring","ar822","ar56","ar_ring","a2a"],"sizes":[1024,16384,65536,262144],"knobs":[{"protocol":"ll"}]}' > gpurun_out/tune_llpack.jsonl 2>&1; python tools/tune.py "{\"scheds\":[\"ag111\",\"ar822\",\"a2a\",\"ring\"],\"sizes\":[1024,16384],\"knobs\":[{\"protocol\":\"ll\"}]}" >> gpurun_out/tune_llpack.jsonl 2>&1
