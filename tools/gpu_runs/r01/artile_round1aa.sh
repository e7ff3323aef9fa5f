# allreduce stage configs under window-major + L2 hints (64/128 MiB)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python tools/tune.py '{"scheds":["ar822","ar56","ar_ring"],"sizes":[67108864,134217728],"knobs":[{},{"tile":32768,"budget":98304},{"tile":49152,"budget":147456},{"tile":65536,"budget":196608},{"tile":32768,"budget":196608}]}' > gpurun_out/tune_artile.jsonl 2>&1
