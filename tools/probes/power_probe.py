#!/usr/bin/env python3
"""Sustained power / clocks of the bench workload against a plain device
copy moving the same DRAM bytes: each runs back to back for `secs` seconds
with NVML sampled every 20 ms; per-launch time (CUDA events) and the median
power / SM clock over the last half are printed as JSON lines."""
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import pynvml  # noqa: E402
import torch  # noqa: E402

from paper_2008_08708_b200 import sccl  # noqa: E402
from paper_2008_08708_b200 import schedules as S  # noqa: E402


def sustained(name, fn, secs, h):
    rows, stop = [], threading.Event()

    def samp():
        while not stop.is_set():
            rows.append((time.perf_counter(), pynvml.nvmlDeviceGetPowerUsage(h) / 1e3,
                         pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                         pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
            stop.wait(0.02)
    th = threading.Thread(target=samp, daemon=True)
    time.sleep(2.0)
    th.start()
    t0 = time.perf_counter()
    times = []
    while time.perf_counter() - t0 < secs:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(4):
            fn()
        b.record()
        b.synchronize()
        times.append((time.perf_counter() - t0, a.elapsed_time(b) / 4 * 1e3))
    stop.set()
    th.join()
    half = [r for r in rows if r[0] - t0 > secs / 2]
    first = [t for s, t in times if s < 0.1]
    last = [t for s, t in times if s > secs / 2]
    print(json.dumps({"what": name, "us_first_100ms": round(statistics.median(first), 1) if first else None,
                      "us_second_half": round(statistics.median(last), 1),
                      "power_w_median": round(statistics.median(r[1] for r in half), 1),
                      "sm_mhz_median": statistics.median(r[2] for r in half),
                      "power_capped_frac": round(sum(1 for r in half if r[3] & 0x4) / max(1, len(half)), 2)}),
          flush=True)


def main():
    secs = float(sys.argv[1]) if len(sys.argv) > 1 else 4.0
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    P, m = 8, 128 << 20
    js = S.to_json(S.hamiltonian_allgather(P))
    plan = sccl.LoopbackPlan(js, m, sccl.U8, device=0)
    send = [torch.randint(0, 256, (m,), dtype=torch.uint8, device="cuda") for _ in range(P)]
    recv = [torch.empty(P * m, dtype=torch.uint8, device="cuda") for _ in range(P)]
    torch.cuda.synchronize()
    sustained("ag777_128MiB", lambda: plan.launch(send, recv), secs, h)
    if len(sys.argv) > 2 and sys.argv[2] == "all":
        for nm, sj, mm, dt in (("ag111_128MiB", S.to_json(S.one_shot_allgather(P)), m, sccl.U8),
                               ("a2a881_512MiB", S.to_json(S.direct_alltoall(P)), 512 << 20, sccl.U8),
                               ("ar822_bf16_256MiB", S.allreduce_from(S.one_shot_allgather(P)), 256 << 20, sccl.BF16)):
            pl = sccl.LoopbackPlan(sj, mm, dt, device=0)
            sd = [torch.randint(0, 256, (mm,), dtype=torch.uint8, device="cuda") for _ in range(P)]
            rc = [torch.empty(pl.recv_bytes, dtype=torch.uint8, device="cuda") for _ in range(P)]
            sustained(nm, lambda: pl.launch(sd, rc), secs, h)
            pl.check()
            pl.close()
            del sd, rc
    # a plain copy with the same DRAM bytes: 4.83 GB read + 4.83 GB written
    n = 4831838208
    src = torch.empty(n, dtype=torch.uint8, device="cuda")
    dst = torch.empty(n, dtype=torch.uint8, device="cuda")
    src.zero_()
    sustained("torch_copy_4.8GB_zeros", lambda: dst.copy_(src), secs, h)
    src.random_(0, 256)
    sustained("torch_copy_4.8GB_random", lambda: dst.copy_(src), secs, h)
    # write-heavy mix like the allgather: 1 GiB read, 8 GiB written (fan-out copies)
    x = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
    x.random_(0, 256)
    ys = [torch.empty(1 << 30, dtype=torch.uint8, device="cuda") for _ in range(8)]

    def fan():
        for y in ys:
            y.copy_(x)
    sustained("torch_copy_fanout_1r8w_GiB_random", fan, secs, h)
    for y in ys:
        y.zero_()
    sendz = [torch.zeros(m, dtype=torch.uint8, device="cuda") for _ in range(P)]
    sustained("ag777_128MiB_zero_payload", lambda: plan.launch(sendz, recv), secs, h)
    plan.check()


if __name__ == "__main__":
    main()
