# BASELINE config 5 (Pareto frontiers at P=2/4/8, loopback) with the multi-storer kernel
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python tools/pareto_sweep.py > gpurun_out/pareto_loopback.jsonl 2> gpurun_out/pareto.err
