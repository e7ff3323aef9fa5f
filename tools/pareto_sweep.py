#!/usr/bin/env python3
"""BASELINE config 5 on one GPU: every committed Pareto-frontier allgather
(paper_2008_08708_b200/frontiers/) and its allreduce (invert + compose) timed in
loopback across sizes (CUDA-graph timed), then an alpha-beta fit per P
(costmodel.fit) and the per-size winner.  One JSON line per measurement,
then one summary line per P."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import torch  # noqa: E402

from paper_2008_08708_b200 import costmodel, sccl  # noqa: E402
from tune import time_plan  # noqa: E402

SIZES = [1 << k for k in range(10, 31, 2)]  # 1 KiB .. 1 GiB per rank (BASELINE config 5 uses config 2/3 sizes)


def main():
    d = os.path.join(ROOT, "paper_2008_08708_b200", "frontiers")
    index = json.load(open(os.path.join(d, "index.json")))
    seen = set()
    maxb = max(SIZES)
    send = [torch.randint(0, 256, (maxb,), dtype=torch.uint8, device="cuda") for _ in range(8)]
    recv = [torch.empty(8 * maxb, dtype=torch.uint8, device="cuda") for _ in range(8)]
    results = []
    for e in index:
        key = (e["topology"], e["C"], e["S"], e["R"])
        if key in seen:
            continue
        seen.add(key)
        ag = open(os.path.join(d, e["file"])).read().strip()
        ar = sccl.compose_allreduce(sccl.invert(ag), ag)
        P = e["P"]
        for coll, js, dt in (("allgather", ag, sccl.U8), ("allreduce", ar, sccl.BF16)):
            for sz in SIZES:
                plan = sccl.LoopbackPlan(js, sz, dt, device=0)
                us = time_plan(plan, [x[:sz] for x in send[:P]], [x[:plan.recv_bytes] for x in recv[:P]],
                               20 if sz >= (1 << 22) else 50)
                busb = (P - 1) * sz if coll == "allgather" else 2 * (P - 1) * sz // P
                r = {"P": P, "collective": coll, "topology": e["topology"], "k": e["k"],
                     "C": e["C"] * (P if coll == "allreduce" else 1), "S": e["S"] * (2 if coll == "allreduce" else 1),
                     "R": e["R"] * (2 if coll == "allreduce" else 1), "bytes_per_rank": sz, "us": round(us, 2),
                     "busbw_per_rank_GBps": round(busb / (us * 1e-6) / 1e9, 2), "protocol": plan.info()["protocol"]}
                results.append(r)
                print(json.dumps(r), flush=True)
                plan.close()
    for P in (2, 4, 8):
        for coll in ("allgather", "allreduce"):
            rows = [r for r in results if r["P"] == P and r["collective"] == coll]
            if not rows:
                continue
            pts = [(r["S"], r["R"], r["C"], r["bytes_per_rank"], r["us"] * 1e-6) for r in rows]
            alpha, beta = costmodel.fit(pts)
            win = {}
            for sz in SIZES:
                best = min((r for r in rows if r["bytes_per_rank"] == sz), key=lambda r: r["us"])
                win[sz] = f"{best['topology']} ({best['C']},{best['S']},{best['R']}) {best['us']}us"
            print(json.dumps({"summary": True, "P": P, "collective": coll, "alpha_us": round(alpha * 1e6, 3),
                              "beta_ps_per_byte": round(beta * 1e12, 3), "winner_per_size": win}), flush=True)


if __name__ == "__main__":
    main()
