# signaler variants (SCCL_SIG_MODE bit0: no idle sleep, bit1: st.release per counter): hop trace + sweep points
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for mode in 0 1 2 3; do
  echo "mode $mode" >> gpurun_out/sig_trace.txt
  SCCL_SIG_MODE=$mode python tools/probes/trace_hops.py 16384:1 262144:8 1048576:32 >> gpurun_out/sig_trace.txt 2>&1
  SCCL_SIG_MODE=$mode python tools/tune.py '{"scheds":["ag777","ring","ar56","ar_ring","ar822","ag111"],"sizes":[262144,1048576,4194304,16777216,134217728],"knobs":[{"protocol":"simple"}]}' > gpurun_out/sig_tune_$mode.jsonl 2>&1
done
