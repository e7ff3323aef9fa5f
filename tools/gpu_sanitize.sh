# compute-sanitizer on the executor: default plans, then window-major + L2 hints forced at small sizes
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_cases.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_summary.txt
  SCCL_WINDOW=4096 SCCL_L2HINT=1 timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_cases.py > gpurun_out/sanitize_${tool}_window.log 2>&1
  echo "$tool window rc=$?" >> gpurun_out/sanitize_summary.txt
done
