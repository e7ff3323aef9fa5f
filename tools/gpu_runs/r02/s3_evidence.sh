# round 2 session 3: evidence with the final session-3 build -- smoke, ncu of the bench kernel, launch list, fuzz, bench N=1 and the reference arm
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/s3e_smoke.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:exec_kernel -s 4 -c 1 -o gpurun_out/s3_prof_ag777 python bench.py --steps 2 --warmup 3 --no-sweep --cpu-seconds 0.1 --cpu-bytes 65536 > gpurun_out/s3_ncu_ag777.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file gpurun_out/s3_launches_bench.csv python bench.py --steps 3 --warmup 3 --no-sweep --cpu-seconds 0.2 --cpu-bytes 65536 > gpurun_out/s3_ncu_launch_bench.log 2>&1
timeout 900 python tools/fuzz_stress.py 400 > gpurun_out/s3_fuzz.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/s3e_bench_ref.log 2>&1
timeout 900 python bench.py > gpurun_out/s3e_bench.log 2>&1
tail -2 gpurun_out/s3_fuzz.log; tail -c 400 gpurun_out/s3e_bench.log
