#!/usr/bin/env python3
"""HBM read/write mix probe on one B200: copy (1R:1W), fill (0R:1W), sum
(1R:0W) and a 1R:8W broadcast copy, CUDA-event timed.  Tells whether the
fan-out ops (AG (1,1,1) writes 8 bytes per byte read) have a lower ceiling
than the 1:1 copy peak in MEASURED_PEAKS.json."""
import json
import torch

N = 2 << 30
a = torch.empty(N, dtype=torch.uint8, device="cuda").fill_(3)
b = torch.empty(N, dtype=torch.uint8, device="cuda")
outs = [torch.empty(N // 8, dtype=torch.uint8, device="cuda") for _ in range(8)]


def t(fn, it=10):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(it):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / it * 1e-3


res = {}
dt = t(lambda: b.copy_(a))
res["copy_1r1w_GBps"] = round(2 * N / dt / 1e9, 1)
dt = t(lambda: b.fill_(7))
res["fill_0r1w_GBps"] = round(N / dt / 1e9, 1)
a32 = a.view(torch.int32)
dt = t(lambda: a32.sum())
res["sum_1r0w_GBps"] = round(N / dt / 1e9, 1)
src = a[:N // 8]
def bc():
    for o in outs:
        o.copy_(src)
dt = t(bc)
res["8_copies_of_one_src_GBps"] = round(16 * (N // 8) / dt / 1e9, 1)
print(json.dumps(res))
