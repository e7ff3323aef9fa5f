#!/usr/bin/env python3
"""Burst vs sustained per-launch time of the bench workload ((7,7,7) AG,
8 x 128 MiB loopback): graph-timed right after plan creation, then
event-timed launches after soaks of increasing length, with nvidia-smi
power / clocks sampled around each point.  One JSON line per point."""
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2008_08708_b200 import sccl  # noqa: E402
from paper_2008_08708_b200 import schedules as S  # noqa: E402


def smi():
    q = "power.draw,clocks.sm,clocks.mem,temperature.gpu,temperature.memory,clocks_throttle_reasons.active"
    out = subprocess.run(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits", "-i", "0"],
                         capture_output=True, text=True).stdout.strip()
    return out


def main():
    m = int(sys.argv[1]) if len(sys.argv) > 1 else 128 << 20
    kc = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    kb = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    P = 8
    js = S.to_json(S.hamiltonian_allgather(P))
    plan = sccl.LoopbackPlan(js, m, sccl.U8, device=0, nchannels=kb, chunk_groups=kc)
    send = [torch.randint(0, 256, (m,), dtype=torch.uint8, device="cuda") for _ in range(P)]
    recv = [torch.empty(P * m, dtype=torch.uint8, device="cuda") for _ in range(P)]
    st = torch.cuda.Stream()
    torch.cuda.synchronize()

    def timed(n):
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
        for a, b in ev:
            a.record(st)
            plan.launch(send, recv, st)
            b.record(st)
        st.synchronize()
        ts = [a.elapsed_time(b) * 1e3 for a, b in ev]
        return sum(ts) / n, min(ts), max(ts)

    time.sleep(2.0)  # let the GPU cool from setup
    print(json.dumps({"point": "idle", "smi": smi()}), flush=True)
    for soak in (0.0, 0.3, 1.0, 3.0, 6.0):
        t0 = time.perf_counter()
        while time.perf_counter() - t0 < soak:
            for _ in range(8):
                plan.launch(send, recv, st)
            st.synchronize()
        s_before = smi()
        avg, mn, mx = timed(20)
        print(json.dumps({"point": f"after {soak}s soak", "kc": plan.info()["chunk_groups"],
                          "kb": plan.info()["byte_parts"], "us_avg": round(avg, 1), "us_min": round(mn, 1),
                          "us_max": round(mx, 1), "smi_before": s_before, "smi_after": smi()}), flush=True)
        time.sleep(3.0)
    plan.check()


if __name__ == "__main__":
    main()
