#!/usr/bin/env python3
"""PCIe ceiling of the e2e path on one B200: pinned host <-> device copy
bandwidth for H2D alone, D2H alone and both at once (1 GiB each), and the
same with each direction split over 4 streams.  The bench's e2e number is
bounded by the concurrent figure (1 GiB in + 1 GiB out per step)."""
import json

import torch

N = 1 << 30
h_in = torch.empty(N, dtype=torch.uint8, pin_memory=True)
h_out = torch.empty(N, dtype=torch.uint8, pin_memory=True)
d_in = torch.empty(N, dtype=torch.uint8, device="cuda")
d_out = torch.empty(N, dtype=torch.uint8, device="cuda")


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e-3


s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
ss = [torch.cuda.Stream() for _ in range(8)]


def h2d():
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)


def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s2)


def both():
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


def both_split(k=4):
    c = N // k
    for i in range(k):
        with torch.cuda.stream(ss[i]):
            d_in[i * c:(i + 1) * c].copy_(h_in[i * c:(i + 1) * c], non_blocking=True)
        with torch.cuda.stream(ss[k + i]):
            h_out[i * c:(i + 1) * c].copy_(d_out[i * c:(i + 1) * c], non_blocking=True)
    for s in ss:
        torch.cuda.current_stream().wait_stream(s)


res = {"h2d_GBps": N / timed(h2d) / 1e9, "d2h_GBps": N / timed(d2h) / 1e9}
t = timed(both)
res["concurrent_each_GBps"] = N / t / 1e9
t = timed(both_split)
res["concurrent_split4_each_GBps"] = N / t / 1e9
print(json.dumps({k: round(v, 1) for k, v in res.items()}))
