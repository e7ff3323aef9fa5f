# round 2: pull lowering -- GPU parity (full suite) + AR timing pull vs push
set -x
nvidia-smi -L; free -g | head -2; nproc
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02_smoke.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r02_pytest_gpu.log 2>&1
timeout 900 python tools/tune.py '{"scheds":["ar822","ar56","ar_ring"],"sizes":[67108864,1048576,65536],"knobs":[{"pull":"off"},{}]}' > gpurun_out/r02_tune_pull.jsonl 2>&1
timeout 900 python tools/tune.py '{"scheds":["ar822"],"sizes":[67108864,268435456],"knobs":[{"tile":65536,"budget":196608},{"tile":32768,"budget":196608},{"tile":16384,"budget":98304},{"tile":65536,"budget":131072},{"tile":49152,"budget":147456},{"tile":32768,"budget":98304,"kb":36},{"tile":32768,"budget":98304,"kb":18}]}' >> gpurun_out/r02_tune_pull.jsonl 2>&1
