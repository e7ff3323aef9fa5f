# round 2 session 3: compute-sanitizer memcheck / synccheck on the multi-process LL path (parity slot sets) and the single-process case set
set -x
make -s -j8 all > /dev/null
for tool in memcheck synccheck; do
  timeout 1200 python tools/sanitize_multiproc.py $tool 6 > gpurun_out/s3_sanitize_mp_$tool.log 2>&1; echo "mp $tool rc=$?" >> gpurun_out/s3_sanitize_summary.txt
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_cases.py > gpurun_out/s3_sanitize_$tool.log 2>&1; echo "cases $tool rc=$?" >> gpurun_out/s3_sanitize_summary.txt
done
cat gpurun_out/s3_sanitize_summary.txt; grep -h "ERROR SUMMARY" gpurun_out/s3_sanitize_*.log
