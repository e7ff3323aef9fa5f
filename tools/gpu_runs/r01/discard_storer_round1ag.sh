# receipt discards issued by the storer warps (overlapping write completion) vs previous build (compute warps)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for i in 1 2; do
for d in 0 1; do
SCCL_DISCARD=$d SCCL_LIB=$PWD/build/ab/libsccl_exec_head.so timeout 600 python tools/tune.py '{"scheds":["ar822","ar56","ar_ring"],"sizes":[67108864,134217728],"knobs":[{}]}' > gpurun_out/tune_dst_head_d${d}_$i.jsonl 2>&1
SCCL_DISCARD=$d timeout 600 python tools/tune.py '{"scheds":["ar822","ar56","ar_ring"],"sizes":[67108864,134217728],"knobs":[{}]}' > gpurun_out/tune_dst_new_d${d}_$i.jsonl 2>&1
done
done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "window_major or counter_release or large or full_sizes" > gpurun_out/pytest_dst.log 2>&1
