# round 2 session 3: final build -- smoke, GPU suite, ncu of the bench kernel + AR captures, launch list, fuzz, bench N=1 + reference arm
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/s3f_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -rs > gpurun_out/s3f_pytest_gpu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:exec_kernel -s 4 -c 1 -o gpurun_out/s3f_prof_ag777 python bench.py --steps 2 --warmup 3 --no-sweep --cpu-seconds 0.1 --cpu-bytes 65536 > gpurun_out/s3f_ncu_ag777.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:exec_kernel -s 3 -c 1 -o gpurun_out/s3f_prof_ar822 python tools/tune.py '{"scheds":["ar822"],"sizes":[67108864],"knobs":[{}]}' > gpurun_out/s3f_ncu_ar822.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:exec_kernel -s 3 -c 1 -o gpurun_out/s3f_prof_ar56 python tools/tune.py '{"scheds":["ar56"],"sizes":[67108864],"knobs":[{}]}' > gpurun_out/s3f_ncu_ar56.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file gpurun_out/s3f_launches_bench.csv python bench.py --steps 3 --warmup 3 --no-sweep --cpu-seconds 0.2 --cpu-bytes 65536 > gpurun_out/s3f_ncu_launch_bench.log 2>&1
timeout 900 python tools/fuzz_stress.py 400 > gpurun_out/s3f_fuzz.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/s3f_bench_ref.log 2>&1
timeout 900 python bench.py > gpurun_out/s3f_bench.log 2>&1
tail -2 gpurun_out/s3f_pytest_gpu.log; tail -1 gpurun_out/s3f_fuzz.log; tail -c 300 gpurun_out/s3f_bench.log
