# round 2: full GPU suite after pull / abort / registration / policy tables / NVLS / frontier wiring
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02f_smoke.log 2>&1
timeout 600 python -m pytest tests/test_gpu_nvls.py tests/test_gpu_parity.py -k "nvls or 48_6_14 or from_machine or tolerance" -x -q -rs > gpurun_out/r02f_pytest_new.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -rs > gpurun_out/r02f_pytest_gpu.log 2>&1
