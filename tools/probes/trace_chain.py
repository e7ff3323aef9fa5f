#!/usr/bin/env python3
"""Where a CTA's time goes in a streaming loopback launch of the bulk
(simple) protocol, from the kernel's debug event trace
(sccl_debug_set_trace).  Per tile (op, tile) the producer records TR_FLAG
(its input counters reached) and TR_EMPTY (its stage came back), the
compute / storer warps TR_FULL (inputs in smem), TR_READY (stage handed to
the storer) and TR_DONE (writes landed).  Per CTA, summed over its tiles:

  issue       ISSUED(t) - EMPTY(t)   producer issuing the tile's bulk loads
  flag_wait   FLAG(t) - ISSUED(t-1)  producer waiting for upstream receipts
              (split: tiles with a receipt input / without)
  empty_wait  EMPTY(t) - FLAG(t)     producer waiting for a free stage
  load        FULL(t) - EMPTY(t)     bulk loads in flight
  compute     READY(t) - FULL(t)     reduce (copy tiles: ~0)
  store       DONE(t) - READY(t)     bulk store issued -> writes landed

usage: python tools/probes/trace_chain.py <schedule: ar56|ar_ring|ag777> <bytes_per_rank> [dtype]"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2008_08708_b200 import sccl  # noqa: E402
from paper_2008_08708_b200 import schedules as S  # noqa: E402

P, CAP = 8, 4096
TR = {"FLAG": 1, "FULL": 2, "READY": 3, "DONE": 4, "PUB": 5, "EMPTY": 7, "ISSUED": 8}


def schedule(name):
    if name == "ar56":
        return S.allreduce_from(S.hamiltonian_allgather(P)), sccl.BF16
    if name == "ar_ring":
        return S.allreduce_from(S.ring_allgather(P)), sccl.BF16
    if name == "ar822":
        return S.allreduce_from(S.one_shot_allgather(P)), sccl.BF16
    return S.to_json(S.hamiltonian_allgather(P)), sccl.U8


def run(name, m, env_note=""):
    js, dt = schedule(name)
    plan = sccl.LoopbackPlan(js, m, dt, device=0)
    info = plan.info()
    grid = info["grid"]
    recv_bytes = m * P if name.startswith("ag") else m
    send = [torch.randint(0, 256, (m,), dtype=torch.uint8, device="cuda") for _ in range(P)]
    recv = [torch.empty(recv_bytes, dtype=torch.uint8, device="cuda") for _ in range(P)]
    for _ in range(3):
        plan.launch(send, recv)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    plan.launch(send, recv)
    b.record()
    torch.cuda.synchronize()
    untraced_us = a.elapsed_time(b) * 1e3
    buf = torch.zeros(grid * CAP * 2, dtype=torch.int64, device="cuda")
    plan.set_trace(buf, CAP)
    a.record()
    plan.launch(send, recv)
    b.record()
    torch.cuda.synchronize()
    traced_us = a.elapsed_time(b) * 1e3
    plan.set_trace(None)
    plan.check()
    rec = buf.view(grid, CAP, 2).cpu().tolist()
    dump = os.environ.get("TRACE_DUMP")
    if dump:  # raw events of channels 0 and 1 of every rank (CTA b = rank * nch + ch)
        nch = info["nchannels"]
        keep = {f"{lr}:{ch}": rec[lr * nch + ch] for lr in range(P) for ch in (0, 1)}
        with open(dump, "w") as f:
            json.dump({"nch": nch, "ctas": {k: [r for r in v if r[0]] for k, v in keep.items()},
                       "program": info["program"]}, f)
    t0 = min(r[0] for cta in rec for r in cta if r[0])
    tot = {k: [] for k in ("flag_wait", "flag_wait_receipt", "flag_wait_none", "issue", "empty_wait", "load",
                           "compute", "store", "span", "tiles")}
    per_tile = {k: [] for k in ("load", "compute", "store")}
    by_op = {}  # receipt wait per program position (op index within the CTA's program), summed per CTA
    overflow = 0
    for cta in rec:
        ev = {}
        n = 0
        for t, meta in cta:
            if not t:
                continue
            n += 1
            e, op, tile = meta & 0xff, (meta >> 8) & 0xffffff, meta >> 32
            rec_ = ev.setdefault((op, tile & 0x7fffffff), {})
            rec_[e] = t - t0
            if e == TR["FLAG"]:
                rec_["waits"] = bool(tile >> 31)
        overflow += n >= CAP
        keys = sorted(ev, key=lambda k: ev[k].get(TR["FLAG"], 1 << 62))
        keys = [k for k in keys if all(TR[x] in ev[k] for x in ("FLAG", "EMPTY", "ISSUED", "FULL", "READY", "DONE"))]
        if not keys:
            continue
        s = dict.fromkeys(("flag_wait", "flag_wait_receipt", "flag_wait_none", "issue", "empty_wait", "load",
                           "compute", "store"), 0)
        prev_issued = None
        for k in keys:
            e = ev[k]
            if prev_issued is not None:
                w = max(0, e[TR["FLAG"]] - prev_issued)
                s["flag_wait"] += w
                s["flag_wait_receipt" if e.get("waits") else "flag_wait_none"] += w
                by_op.setdefault(k[0], []).append(w)
            s["issue"] += e[TR["ISSUED"]] - e[TR["EMPTY"]]
            s["empty_wait"] += e[TR["EMPTY"]] - e[TR["FLAG"]]
            per_tile["load"].append(e[TR["FULL"]] - e[TR["EMPTY"]])
            per_tile["compute"].append(e[TR["READY"]] - e[TR["FULL"]])
            per_tile["store"].append(e[TR["DONE"]] - e[TR["READY"]])
            s["load"] += per_tile["load"][-1]
            s["compute"] += per_tile["compute"][-1]
            s["store"] += per_tile["store"][-1]
            prev_issued = e[TR["ISSUED"]]
        for k2, v in s.items():
            tot[k2].append(v)
        tot["span"].append(ev[keys[-1]][TR["DONE"]] - ev[keys[0]][TR["FLAG"]])
        tot["tiles"].append(len(keys))
    out = {"schedule": name, "bytes_per_rank": m, "grid": grid, "tile": info["tile_bytes"], "nstage": info["nstage"],
           "window": info["window"], "untraced_us": round(untraced_us, 1), "traced_us": round(traced_us, 1),
           "ctas_overflowed": overflow, "note": env_note}
    out.update({f"cta_{k}_us_median": round(statistics.median(v) / 1e3, 2) for k, v in tot.items() if k != "tiles"})
    out["tiles_per_cta_median"] = statistics.median(tot["tiles"])
    out.update({f"tile_{k}_us_median": round(statistics.median(v) / 1e3, 3) for k, v in per_tile.items()})
    out.update({f"tile_{k}_us_p90": round(sorted(v)[int(0.9 * len(v))] / 1e3, 3) for k, v in per_tile.items()})
    ops = sorted(by_op)
    base = ops[0] if ops else 0
    # mean over CTAs of the wait before each op (all its tiles), in program order
    out["wait_by_op_us"] = [round(sum(by_op[o]) / len(rec) / 1e3, 2) for o in ops]
    out["op_index_base"] = base
    print(json.dumps(out), flush=True)
    plan.close()


if __name__ == "__main__":
    name = sys.argv[1] if len(sys.argv) > 1 else "ar56"
    m = int(sys.argv[2]) if len(sys.argv) > 2 else 64 << 20
    run(name, m, os.environ.get("TRACE_NOTE", ""))
