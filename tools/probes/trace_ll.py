#!/usr/bin/env python3
"""Where a small LL launch spends its time, from the kernel's debug event
trace: per CTA, kernel entry -> epoch known -> op descriptors read -> data
moved (per op) -> exit.  Medians over CTAs, microseconds from the earliest
entry of the launch.  usage: python tools/probes/trace_ll.py"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2008_08708_b200 import sccl  # noqa: E402
from paper_2008_08708_b200 import schedules as S  # noqa: E402

CAP = 64
P = 8
cases = {"null1": S.to_json(S._sched("allgather", "full:1", 1, 1, 1, [1], [])),
         "ag111": S.to_json(S.one_shot_allgather(P)), "ar822": S.allreduce_from(S.one_shot_allgather(P)),
         "ag777": S.to_json(S.hamiltonian_allgather(P))}
for name, js in cases.items():
    Pn = json.loads(js)["P"]
    m = 1024
    plan = sccl.LoopbackPlan(js, m, sccl.U8 if not name.startswith("ar") else sccl.BF16, device=0, protocol="ll")
    grid = plan.info()["grid"]
    send = [torch.randint(0, 256, (m,), dtype=torch.uint8, device="cuda") for _ in range(Pn)]
    recv = [torch.empty(plan.recv_bytes, dtype=torch.uint8, device="cuda") for _ in range(Pn)]
    torch.cuda.synchronize()
    for _ in range(5):
        plan.launch(send, recv)
    torch.cuda.synchronize()
    buf = torch.zeros(grid * CAP * 2, dtype=torch.int64, device="cuda")
    plan.set_trace(buf, CAP)
    plan.launch(send, recv)
    torch.cuda.synchronize()
    plan.set_trace(None)
    rec = buf.view(grid, CAP, 2).cpu().tolist()
    t0 = min(r[0] for cta in rec for r in cta if r[0])
    seg = {"entry": [], "epoch": [], "desc1": [], "d_op": [], "d_in": [], "d_ptr": [], "d_bar": [], "data1": [],
           "ops": [], "exit": []}
    for cta in rec:
        ev = [(t - t0, meta & 0xff) for t, meta in cta if t]
        if not ev:
            continue
        get = lambda e: [t for t, x in ev if x == e]
        st, ep, ds, dn, en = get(0), get(1), get(2), get(4), get(6)
        seg["entry"].append(st[0])
        seg["epoch"].append(ep[0] - st[0])
        e7, e8, e9 = get(7), get(8), get(9)
        if ds and e7 and e8 and e9:
            seg["d_op"].append(e7[0] - ep[0])
            seg["d_in"].append(e8[0] - e7[0])
            seg["d_ptr"].append(e9[0] - e8[0])
            seg["d_bar"].append(ds[0] - e9[0])
        if ds:
            seg["desc1"].append(ds[0] - ep[0])
            seg["data1"].append(dn[0] - ds[0])
            seg["ops"].append(len(ds))
        seg["exit"].append(en[0] - (dn[-1] if dn else ep[0]))
    print(json.dumps({"case": name, "grid": grid, **{k: round(statistics.median(v) / 1e3, 3) if v else None
                                                     for k, v in seg.items()},
                      "span_us": round(max(r[0] for cta in rec for r in cta if r[0]) / 1e3 - t0 / 1e3, 3)}))
    plan.close()
