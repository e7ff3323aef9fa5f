#!/bin/bash
# bisect the back-to-back ag_777 tile=4096 failure: head lib / new lib / new lib without descriptor cache
mkdir -p gpurun_out
T="tests/test_gpu_parity.py::test_back_to_back_launches_advance_epochs"
for i in 1 2 3; do
echo "head $i: $(SCCL_LIB=$PWD/build/ab/libsccl_exec_head.so timeout 120 python -m pytest $T -x -q 2>&1 | tail -1)"
echo "new $i: $(timeout 120 python -m pytest $T -x -q 2>&1 | tail -1)"
echo "new nocache $i: $(SCCL_DCACHE=0 timeout 120 python -m pytest $T -x -q 2>&1 | tail -1)"
done > gpurun_out/bisect.log 2>&1
cat gpurun_out/bisect.log
