#!/usr/bin/env python3
"""Same-box A/B of a plan-creation environment knob on loopback launches:
for each schedule, plans built with knob=A and knob=B are timed alternately
(CUDA events over `iters` back-to-back launches, `reps` alternations); prints
one JSON line per (schedule, size) with both medians.  The knob is read at
plan creation, so both plans live side by side.
usage: python tools/probes/ab_env.py KNOB A B sched:bytes[:dtype] ..."""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2008_08708_b200 import sccl  # noqa: E402
from paper_2008_08708_b200 import schedules as S  # noqa: E402

P = 8
SCHED = {
    "ar56": lambda: (S.allreduce_from(S.hamiltonian_allgather(P)), sccl.BF16, 1),
    "ar56f": lambda: (S.allreduce_from(S.hamiltonian_allgather(P)), sccl.F32, 1),
    "ar_ring": lambda: (S.allreduce_from(S.ring_allgather(P)), sccl.BF16, 1),
    "ar822": lambda: (S.allreduce_from(S.one_shot_allgather(P)), sccl.BF16, 1),
    "ar822f": lambda: (S.allreduce_from(S.one_shot_allgather(P)), sccl.F32, 1),
    "ar_ringf": lambda: (S.allreduce_from(S.ring_allgather(P)), sccl.F32, 1),
    "ag777": lambda: (S.to_json(S.hamiltonian_allgather(P)), sccl.U8, P),
    "ag_ring": lambda: (S.to_json(S.ring_allgather(P)), sccl.U8, P),
    "ag111": lambda: (S.to_json(S.one_shot_allgather(P)), sccl.U8, P),
    "a2a": lambda: (S.to_json(S.direct_alltoall(P)), sccl.U8, 1),
}


def main():
    knob, va, vb = sys.argv[1:4]
    iters, reps = 10, 5
    for spec in sys.argv[4:]:
        name, nb = spec.split(":")[:2]
        nb = int(nb)
        js, dt, mult = SCHED[name]()
        plans = {}
        for v in (va, vb):
            os.environ[knob] = v
            plans[v] = sccl.LoopbackPlan(js, nb, dt, device=0)
        os.environ.pop(knob, None)
        send = [torch.randint(0, 256, (nb,), dtype=torch.uint8, device="cuda") for _ in range(P)]
        outs = {v: [torch.empty(nb * mult, dtype=torch.uint8, device="cuda") for _ in range(P)] for v in (va, vb)}
        t = {va: [], vb: []}
        for _ in range(3):
            for v in (va, vb):
                plans[v].launch(send, outs[v])
        torch.cuda.synchronize()
        graphs = {}
        if os.environ.get("AB_GRAPH") == "1":  # small sizes: time CUDA-graph replays (no host launch cost)
            st = torch.cuda.Stream()
            for v in (va, vb):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=st):
                    for _ in range(iters * 10):
                        plans[v].launch(send, outs[v], st)
                graphs[v] = g
        for _ in range(reps):
            for v in (va, vb):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                if graphs:
                    graphs[v].replay()
                    torch.cuda.synchronize()
                    a.record()
                    graphs[v].replay()
                    b.record()
                    torch.cuda.synchronize()
                    t[v].append(a.elapsed_time(b) * 1e3 / (iters * 10))
                    continue
                a.record()
                for _ in range(iters):
                    plans[v].launch(send, outs[v])
                b.record()
                torch.cuda.synchronize()
                t[v].append(a.elapsed_time(b) * 1e3 / iters)
        for v in (va, vb):
            plans[v].check()
        same = all(torch.equal(x, y) for x, y in zip(outs[va], outs[vb]))
        print(json.dumps({"knob": knob, "schedule": name, "bytes_per_rank": nb, f"us_{va}": round(statistics.median(t[va]), 2),
                          f"us_{vb}": round(statistics.median(t[vb]), 2), "outputs_equal": same,
                          "ratio": round(statistics.median(t[vb]) / statistics.median(t[va]), 4)}), flush=True)
        for v in (va, vb):
            plans[v].close()


if __name__ == "__main__":
    main()
