#!/usr/bin/env python3
"""Small executor cases for compute-sanitizer (memcheck / racecheck /
synccheck): both protocols, copy and fused-reduce programs, aligned and
unaligned sizes, checked against the oracle."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
from paper_2008_08708_b200 import sccl  # noqa: E402
from paper_2008_08708_b200 import schedules as S  # noqa: E402

cases = [
    (S.to_json(S.hamiltonian_allgather(8)), 20000, O.U8, "simple"),
    (S.to_json(S.hamiltonian_allgather(8)), 3000, O.U8, "ll"),
    (S.allreduce_from(S.one_shot_allgather(8)), 40960, O.BF16, "simple"),
    (S.allreduce_from(S.ring_allgather(4)), 1000, O.F32, "ll"),
    (S.to_json(S.direct_alltoall(4, 8)), 4096 + 32, O.U8, "simple"),
    (S.to_json(S.bidir_ring_allgather(8)), 1000, O.U8, "simple"),  # unaligned offsets
    # round 2: pull-lowered reductions (peers' SEND read in place), push for comparison
    (S.allreduce_from(S.hamiltonian_allgather(8)), 65536, O.BF16, "simple"),
    (S.allreduce_from(S.one_shot_allgather(8)), 8192, O.F32, "ll"),
    (S.allreduce_from(S.one_shot_allgather(8)), 40960, O.BF16, "simple", "off"),
    # round 2 session 2: one chunk group, byte parts below a tile (one-shot copy / pulled one-shot reduce)
    (S.to_json(S.one_shot_allgather(8)), 65536 + 48, O.U8, "simple"),
    (S.allreduce_from(S.one_shot_allgather(8)), 1 << 20, O.BF16, "simple"),
]
bad = 0
for js, nb, dt, proto, *pull in cases:
    d = json.loads(js)
    ins = O.seeded_inputs(d["collective"], d["P"], nb, dt, 1)
    ref = O.execute(d, ins, nb, dt)
    plan = sccl.LoopbackPlan(js, nb, dt, device=0, protocol=proto, timeout_ms=120000,
                             pull=pull[0] if pull else "auto")
    send = [torch.from_numpy(x).cuda() for x in ins]
    recv = [torch.zeros(r.size, dtype=torch.uint8, device="cuda") for r in ref]
    plan.launch(send, recv)
    torch.cuda.synchronize()
    ok = all(np.array_equal(a.cpu().numpy(), b) for a, b in zip(recv, ref))
    bad += not ok
    print(d["collective"], proto, nb, "ok" if ok else "MISMATCH", flush=True)
sys.exit(1 if bad else 0)
