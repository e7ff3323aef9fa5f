python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python tools/tune.py '{"scheds":["ar822","ar56","ag777","ag111"],"sizes":[1048576,16777216,134217728],"knobs":[{"order":"canonical"},{"order":"rotate"}]}' > gpurun_out/tune_order.jsonl 2>&1
