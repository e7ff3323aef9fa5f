# round 2: full GPU suite (NVLS gated on a trial multicast team) + compute-sanitizer
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02g_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -rs > gpurun_out/r02g_pytest_gpu.log 2>&1
rm -f gpurun_out/sanitize_summary.txt
bash tools/gpu_sanitize.sh
