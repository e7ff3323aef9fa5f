#!/bin/bash
mkdir -p gpurun_out
T="tests/test_gpu_parity.py::test_back_to_back_launches_advance_epochs"
for v in idle_only item_only; do
echo "$v: $(SCCL_LIB=$PWD/build/ab/libsccl_exec_$v.so timeout 120 python -m pytest $T -x -q 2>&1 | tail -1)"
done > gpurun_out/bisect2.log 2>&1
cat gpurun_out/bisect2.log
