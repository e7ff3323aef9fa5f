#!/usr/bin/env python3
"""Per-hop latency breakdown of the bulk (simple) protocol from the kernel's
debug event trace (sccl_debug_set_trace).  For a ring allgather every op at
rank r, step s >= 1 forwards the receipt rank r-1 published at step s-1, so

  hop      = t_flag(r, s) - t_pub(r-1, s-1)   counter published -> consumer saw it
  load     = t_full - t_flag                  bulk load issued -> data in smem
  pass     = t_ready - t_full                 compute warps hand the stage on
  store    = t_done - t_ready                 bulk store issued -> writes landed
  signal   = t_pub - t_done                   completion ring -> counter stored

Medians over ranks, steps and channels (first tile of each op; last tile for
t_pub).  usage: python tools/probes/trace_hops.py [bytes_per_rank ...]"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2008_08708_b200 import sccl  # noqa: E402
from paper_2008_08708_b200 import schedules as S  # noqa: E402

P, CAP = 8, 512


def run(m, kb):
    js = S.to_json(S.ring_allgather(P))
    plan = sccl.LoopbackPlan(js, m, sccl.U8, device=0, protocol="simple", nchannels=kb, chunk_groups=1)
    info = plan.info()
    grid, nch = info["grid"], info["nchannels"]
    send = [torch.randint(0, 256, (m,), dtype=torch.uint8, device="cuda") for _ in range(P)]
    recv = [torch.empty(P * m, dtype=torch.uint8, device="cuda") for _ in range(P)]
    for _ in range(3):
        plan.launch(send, recv)
    torch.cuda.synchronize()
    buf = torch.zeros(grid * CAP * 2, dtype=torch.int64, device="cuda")
    plan.set_trace(buf, CAP)
    plan.launch(send, recv)
    torch.cuda.synchronize()
    plan.set_trace(None)
    plan.check()
    want = torch.cat(send)
    assert all(torch.equal(r, want) for r in recv)
    rec = buf.view(grid, CAP, 2).cpu().tolist()
    # per (rank, channel): op order = step order (ring: one op per step, then the wait)
    ev = {}
    t0 = min(r[0] for cta in rec for r in cta if r[0])
    for b, cta in enumerate(rec):
        lr, ch = divmod(b, nch)
        for t, meta in cta:
            if not t:
                continue
            e, op, tile = meta & 0xff, (meta >> 8) & 0xffffff, meta >> 32
            ev.setdefault((lr, ch), []).append((t - t0, e, op, tile))
    seg = {k: [] for k in ("hop", "load", "pass", "store", "signal", "step", "sig_wake", "sig_loads", "sig_fence")}
    for (lr, ch), L in ev.items():
        ops = sorted({op for _, e, op, _ in L if e in (1, 2, 3, 4, 5)})
        first = lambda e, op: min((t for t, x, o, _ in L if x == e and o == op), default=None)
        last = lambda e, op: max((t for t, x, o, _ in L if x == e and o == op), default=None)
        for i, o in enumerate(ops):
            dn, w, ld, pb = first(4, o), first(7, o), first(8, o), first(5, o)
            if None not in (dn, w, ld, pb):
                seg["sig_wake"].append(w - dn)
                seg["sig_loads"].append(ld - w)
                seg["sig_fence"].append(pb - ld)
        ev[(lr, ch)] = {"ops": ops, "flag": [first(1, o) for o in ops], "full": [first(2, o) for o in ops],
                        "ready": [first(3, o) for o in ops], "done": [first(4, o) for o in ops],
                        "pub": [last(5, o) for o in ops]}
        d = ev[(lr, ch)]
        for i in range(len(ops)):
            if None in (d["flag"][i], d["full"][i], d["ready"][i], d["done"][i]):
                continue
            seg["load"].append(d["full"][i] - d["flag"][i])
            seg["pass"].append(d["ready"][i] - d["full"][i])
            seg["store"].append(d["done"][i] - d["ready"][i])
            if d["pub"][i] is not None:
                seg["signal"].append(d["pub"][i] - d["done"][i])
            if i:
                seg["step"].append(d["flag"][i] - d["flag"][i - 1])
    for (lr, ch), d in ev.items():
        prev = ev.get(((lr - 1) % P, ch))
        if not prev:
            continue
        for s in range(1, min(len(d["ops"]), len(prev["ops"]))):
            if d["flag"][s] is not None and prev["pub"][s - 1] is not None:
                seg["hop"].append(d["flag"][s] - prev["pub"][s - 1])
    out = {"bytes_per_rank": m, "grid": grid, "nchannels": nch, "tile": info["tile_bytes"]}
    out.update({k: round(statistics.median(v), 0) if v else None for k, v in seg.items()})
    out["n"] = len(seg["hop"])
    print(json.dumps(out), flush=True)
    plan.close()


if __name__ == "__main__":
    for arg in (sys.argv[1:] or ["16384:1", "262144:8", "1048576:32"]):
        m, kb = (int(x) for x in arg.split(":"))
        run(m, kb)
