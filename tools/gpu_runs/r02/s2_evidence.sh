# round 2 session 2: evidence after the policy changes -- smoke, ncu of the bench kernel and the 64 MiB
# pulled allreduce, launch list with DRAM bytes, sanitizer, bench N=1 and the reference arm
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/s2e_smoke.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:exec_kernel -s 4 -c 1 -o gpurun_out/s2_prof_ag777 python bench.py --steps 2 --warmup 3 --no-sweep --cpu-seconds 0.1 --cpu-bytes 65536 > gpurun_out/s2_ncu_ag777.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:exec_kernel -s 3 -c 1 -o gpurun_out/s2_prof_ar822 python tools/tune.py '{"scheds":["ar822"],"sizes":[67108864],"knobs":[{}]}' > gpurun_out/s2_ncu_ar822.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file gpurun_out/s2_launches_bench.csv python bench.py --steps 3 --warmup 3 --no-sweep --cpu-seconds 0.2 --cpu-bytes 65536 > gpurun_out/s2_ncu_launch_bench.log 2>&1
rm -f gpurun_out/sanitize_summary.txt
bash tools/gpu_sanitize.sh
timeout 900 python bench.py --impl reference > gpurun_out/s2e_bench_ref.log 2>&1
timeout 900 python bench.py > gpurun_out/s2e_bench.log 2>&1
cat gpurun_out/sanitize_summary.txt
tail -c 600 gpurun_out/s2e_bench.log
