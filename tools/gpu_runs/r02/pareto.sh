# round 2: BASELINE config 5 sweep -- every committed frontier (ring / full / switch at P = 2, 4, 8), AG + AR, 1 KiB - 1 GiB
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 2400 python tools/pareto_sweep.py > gpurun_out/r02_pareto_sweep.jsonl 2> gpurun_out/r02_pareto_sweep.err
