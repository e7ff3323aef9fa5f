# round 2: cooperative abort, registered buffers, multidevice harness (shared GPU), AR pull grid
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02b_smoke.log 2>&1
timeout 600 python -m pytest tests/test_gpu_watchdog.py tests/test_gpu_multiprocess.py tests/test_gpu_multidevice.py -x -q -rs > gpurun_out/r02b_pytest_mp.log 2>&1
SCCL_MULTIDEVICE_SHARE=1 SCCL_MULTIDEVICE_WORLD=2 timeout 900 python -m pytest tests/test_gpu_multidevice.py -x -q > gpurun_out/r02b_multidevice_share.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r02b_pytest_gpu.log 2>&1
timeout 900 python tools/tune.py '{"scheds":["ar822"],"sizes":[67108864,16777216,268435456],"knobs":[{"kb":18},{"kb":9},{"kb":12},{"kb":24},{"tile":16384,"budget":98304,"kb":18},{"tile":49152,"budget":147456,"kb":18},{"tile":65536,"budget":196608,"kb":9},{"tile":32768,"budget":196608,"kb":18}]}' > gpurun_out/r02b_tune_ar822.jsonl 2>&1
