#!/usr/bin/env python3
"""BASELINE configs 1-4 as size sweeps on one B200 (8 loopback ranks), one
JSON line per (config, schedule, dtype, size):

  cfg1  ring(8) latency-optimal allgathers (1,4,4) and (2,4,7) at 1 MiB/rank:
        the CPU reference executor (oracle, 1 thread and all threads) and
        the GPU executor on the same schedule file
  cfg2  allgather (7,7,7), (1,1,1), ring (1,7,7), 1 KiB - 1 GiB per rank
  cfg3  allreduce (8,2,2), (56,14,14), ring (8,14,14), bf16 and f32,
        1 KiB - 1 GiB per rank
  cfg4  alltoall (8,1,1), 64 KiB - 256 MiB per rank

GPU times: K launches captured in one CUDA graph, CUDA events around the
replay (host launch cost excluded), after 3 warm-up launches; no L2 flush
(sizes < 126 MB are L2-resident between launches, as in nccl-tests).
busbw per rank follows nccl-tests: AG (P-1)m, AR 2(P-1)/P M, A2A (P-1)/P M.
hbm_frac = algorithmic HBM bytes of the lowered program / t / measured peak
(can pass 1: window-major execution re-reads relayed receipts from L2);
frac_of_min = (inputs read once + outputs written once) / t / peak.

usage: python tools/size_sweep.py [cfg1,cfg2,cfg3,cfg4] [--max-log2 N]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import torch  # noqa: E402

from paper_2008_08708_b200 import sccl  # noqa: E402
from paper_2008_08708_b200 import schedules as S  # noqa: E402
from tune import time_plan  # noqa: E402

P = 8
GOLD = os.path.join(ROOT, "tests", "golden", "schedules")


def peak_gbs():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        return 6650.0


def hbm_bytes(plan):
    prog = plan.info()["program"]
    return sum(op["len"] * (len(op["ins"]) + len(op["outs"])) for rk in prog["ranks"] for op in rk["ops"]
               if op["kind"] != "wait")


def busbytes(coll, m):
    if coll == "allgather":
        return (P - 1) * m
    if coll == "allreduce":
        return 2 * (P - 1) * m // P
    return (P - 1) * m // P  # alltoall


def iters_for(sz):
    return 5 if sz >= (256 << 20) else 20 if sz >= (4 << 20) else 100


def gpu_sweep(cfg, coll, scheds, dtypes, sizes):
    maxb = max(sizes)
    recv_mult = P if coll == "allgather" else 1
    send = [torch.randint(0, 256, (maxb,), dtype=torch.uint8, device="cuda") for _ in range(P)]
    recv = [torch.empty(recv_mult * maxb, dtype=torch.uint8, device="cuda") for _ in range(P)]
    pk = peak_gbs()
    for name, js in scheds:
        for dt, dtn in dtypes:
            for sz in sizes:
                row = {"cfg": cfg, "collective": coll, "schedule": name, "dtype": dtn, "bytes_per_rank": sz,
                       "total_bytes": P * sz}  # nccl-tests' size convention (all ranks)
                try:
                    plan = sccl.LoopbackPlan(js, sz, dt, device=0)
                except sccl.SCCLError as e:
                    row["error"] = str(e)[:160]
                    print(json.dumps(row), flush=True)
                    continue
                us = time_plan(plan, [x[:sz] for x in send], [x[:plan.recv_bytes] for x in recv], iters_for(sz))
                info = plan.info()
                hb = hbm_bytes(plan)
                mn = P * sz + P * P * sz if coll == "allgather" else 2 * P * sz  # inputs once + outputs once
                row.update({"us": round(us, 2), "busbw_per_rank_GBps": round(busbytes(coll, sz) / us / 1e3, 2),
                            "hbm_GBps": round(hb / us / 1e3, 1), "hbm_frac": round(hb / us / 1e3 / pk, 3),
                            "frac_of_min": round(mn / us / 1e3 / pk, 3),
                            "protocol": info["protocol"], "grid": info["grid"], "tile": info["tile_bytes"],
                            "nstage": info["nstage"]})
                print(json.dumps(row), flush=True)
                plan.close()
    del send, recv
    torch.cuda.empty_cache()


def cfg1():
    """CPU reference executor vs the GPU executor on ring(8) (1,4,4) and the
    synthesized (2,4,7), 1 MiB per rank (BASELINE config 1)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    m = 1 << 20
    scheds = [("ring8 (1,4,4) bidirectional", S.to_json(S.bidir_ring_allgather(P))),
              ("ring8 (2,4,7) synthesized", open(os.path.join(GOLD, "ag_ring8_2_4_7.json")).read().strip())]
    cores = os.cpu_count() or 1
    for name, js in scheds:
        d = json.loads(js)
        ins = O.seeded_inputs(d["collective"], P, m, O.U8, 0)
        for th in sorted({1, cores}):
            ex = O.Execution(d, ins, m, O.U8, check=True)
            ex.run(th)
            times = []
            t_end = time.perf_counter() + 3.0
            while time.perf_counter() < t_end or len(times) < 20:
                t0 = time.perf_counter()
                ex.run(th)
                times.append(time.perf_counter() - t0)
            times.sort()
            med = times[len(times) // 2]
            print(json.dumps({"cfg": "cfg1", "impl": "cpu_reference", "schedule": name, "threads": th,
                              "bytes_per_rank": m, "runs": len(times), "us_median": round(med * 1e6, 1),
                              "us_min": round(times[0] * 1e6, 1),
                              "busbw_per_rank_GBps": round((P - 1) * m / med / 1e9, 3)}), flush=True)
    gpu_sweep("cfg1", "allgather", scheds, [(sccl.U8, "u8")], [m])


def main():
    which = sys.argv[1].split(",") if len(sys.argv) > 1 and not sys.argv[1].startswith("-") else \
        ["cfg1", "cfg2", "cfg3", "cfg4"]
    maxlog = int(sys.argv[sys.argv.index("--max-log2") + 1]) if "--max-log2" in sys.argv else 30
    big = [1 << k for k in range(10, maxlog + 1, 2)]
    ag = S.hamiltonian_allgather(P)
    if "cfg1" in which:
        cfg1()
    if "cfg2" in which:
        gpu_sweep("cfg2", "allgather",
                  [("(7,7,7) hamiltonian full:8", S.to_json(ag)),
                   ("(1,1,1) one-shot full:8", S.to_json(S.one_shot_allgather(P))),
                   ("(1,7,7) ring:8", S.to_json(S.ring_allgather(P)))],
                  [(sccl.U8, "u8")], big)
    if "cfg3" in which:
        gpu_sweep("cfg3", "allreduce",
                  [("(8,2,2) one-shot RS+AG", S.allreduce_from(S.one_shot_allgather(P))),
                   ("(56,14,14) hamiltonian RS+AG", S.allreduce_from(ag)),
                   ("(8,14,14) ring RS+AG", S.allreduce_from(S.ring_allgather(P)))],
                  [(sccl.BF16, "bf16"), (sccl.F32, "f32")], big)
    if "cfg4" in which:
        gpu_sweep("cfg4", "alltoall", [("(8,1,1) direct full:8", S.to_json(S.direct_alltoall(P)))],
                  [(sccl.U8, "u8")], [1 << k for k in range(16, min(maxlog, 28) + 1, 2)])


if __name__ == "__main__":
    main()
