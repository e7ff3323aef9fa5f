# round 2 session 2: bench timed region with the in-process NVML sampler vs nvidia-smi subprocesses
for i in 1 2; do
  python bench.py --no-sweep --cpu-seconds 1 > gpurun_out/s2_ab_nvml_$i.log 2>&1
  SCCL_BENCH_SMI=1 python bench.py --no-sweep --cpu-seconds 1 > gpurun_out/s2_ab_smi_$i.log 2>&1
done
for f in gpurun_out/s2_ab_*.log; do python -c "
import json,sys
l=[x for x in open('$f') if x.startswith('{')][-1]; d=json.loads(l)
print('$f', d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac'], d['clocks'])"; done
