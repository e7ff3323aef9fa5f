python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python tools/size_sweep.py > gpurun_out/size_sweep.jsonl 2> gpurun_out/size_sweep.err
nproc > gpurun_out/nproc.txt; lscpu > gpurun_out/lscpu.txt
