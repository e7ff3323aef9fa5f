# round 2 session 3: final evidence after the LL ok-flag, prologue fastdiv and barrier changes -- smoke, GPU suite, ncu of the bench kernel, launch list, size sweep, fuzz, bench N=1 + reference arm
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/s3w_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -rs > gpurun_out/s3w_pytest_gpu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:exec_kernel -s 4 -c 1 -o gpurun_out/s3w_prof_ag777 python bench.py --steps 2 --warmup 3 --no-sweep --cpu-seconds 0.1 --cpu-bytes 65536 > gpurun_out/s3w_ncu_ag777.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file gpurun_out/s3w_launches_bench.csv python bench.py --steps 3 --warmup 3 --no-sweep --cpu-seconds 0.2 --cpu-bytes 65536 > gpurun_out/s3w_ncu_launch_bench.log 2>&1
timeout 2400 python tools/size_sweep.py > gpurun_out/s3w_size_sweep.jsonl 2> gpurun_out/s3w_size_sweep.err
timeout 900 python tools/fuzz_stress.py 400 > gpurun_out/s3w_fuzz.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/s3w_bench_ref.log 2>&1
timeout 900 python bench.py > gpurun_out/s3w_bench.log 2>&1
tail -2 gpurun_out/s3w_pytest_gpu.log; tail -1 gpurun_out/s3w_fuzz.log
