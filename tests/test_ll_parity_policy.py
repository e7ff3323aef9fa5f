"""Host side of the epoch-parity LL slot sets (plan.cpp ll_parity_safe):
which schedules may skip the entry handshake, restated here as a separate
Python check of the same completion-set argument and compared with the
library's choice (host-only plans, no GPU)."""
import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2008_08708_b200 import sccl, schedules as S  # noqa: E402


def completion_safe(js: str) -> bool:
    """Every cross-rank send S -> R: R's launch must be one S's completion
    waited for (a chain of sends of the same chunk, each reading its
    sender's value at the start of its step, from R to S)."""
    d = json.loads(js)
    phases = d["phases"] if "phases" in d else [d]
    P = d["P"]
    dep = {}  # (chunk, node) -> ranks
    done = [set() for _ in range(P)]
    for ph in phases:
        for st in range(ph["S"]):
            new = {k: set(v) for k, v in dep.items()}
            for c, src, dst, step in ph["sends"]:
                if step != st:
                    continue
                m = dep.get((c, src), set()) | {src}
                new.setdefault((c, dst), set()).update(m)
                done[dst] |= m
            dep = new
    return all(dst in done[src] for ph in phases for c, src, dst, step in ph["sends"])


CASES = [
    ("ag_oneshot8", S.to_json(S.one_shot_allgather(8)), sccl.U8, True),
    ("ag_ring8", S.to_json(S.ring_allgather(8)), sccl.U8, True),
    ("ag_ham8", S.to_json(S.hamiltonian_allgather(8)), sccl.U8, True),
    ("ag_bidir8", S.to_json(S.bidir_ring_allgather(8)), sccl.U8, True),
    ("ag_rd4", S.to_json(S.recursive_doubling_ring4()), sccl.U8, True),
    ("a2a8", S.to_json(S.direct_alltoall(8)), sccl.U8, True),
    ("rs_ring4", S.reducescatter_from(S.ring_allgather(4)), sccl.F32, True),
    ("ar_oneshot8", S.allreduce_from(S.one_shot_allgather(8)), sccl.BF16, True),
    ("ar_ham8", S.allreduce_from(S.hamiltonian_allgather(8)), sccl.BF16, True),
    ("bcast8", S.to_json(S.one_shot_broadcast(8)), sccl.U8, False),
    ("bcast_chain4", S.to_json(S.pipelined_chain_broadcast(4, 4)), sccl.U8, False),
    ("gather4", S.to_json(S.direct_gather(4)), sccl.U8, False),
    ("scatter4", S.to_json(S.direct_scatter(4)), sccl.U8, False),
    ("reduce4", S.reduce_from(S.one_shot_broadcast(4)), sccl.I32, False),
]


@pytest.mark.parametrize("name,js,dt,expect", CASES, ids=[c[0] for c in CASES])
def test_ll_parity_choice(name, js, dt, expect):
    assert completion_safe(js) == expect
    P = json.loads(js)["P"]
    ll = sccl.Plan(js, 0, P, 4096 * P, dt, device=-1, protocol="ll")
    assert ll.info()["ll_parity"] == int(expect)
    simple = sccl.Plan(js, 0, P, 4096 * P, dt, device=-1, protocol="simple")
    assert simple.info()["ll_parity"] == 0  # the simple protocol always keeps the handshake
    if expect:  # two slot sets: the region grows by one scratch set
        os.environ["SCCL_LL_PARITY"] = "0"
        try:
            hs = sccl.Plan(js, 0, P, 4096 * P, dt, device=-1, protocol="ll")
        finally:
            os.environ.pop("SCCL_LL_PARITY")
        assert hs.info()["ll_parity"] == 0
        assert ll.info()["region_bytes"] >= hs.info()["region_bytes"]
        assert ll.info()["program"]["fingerprint"] == hs.info()["program"]["fingerprint"]


def test_random_allgathers_are_parity_safe():
    """Every allgather delivers every rank's chunk to every rank, so every
    rank is in every completion set."""
    for seed in range(10):
        js = S.to_json(S.random_allgather(5, 2, 3, seed=seed))
        assert completion_safe(js)


def test_bind_refuses_mixed_parity():
    """A rank built with SCCL_LL_PARITY=0 cannot bind with ranks that use the
    parity slot sets (the region sizes can round to the same 2 MiB)."""
    js = S.to_json(S.one_shot_allgather(2))
    a = sccl.Plan(js, 0, 2, 4096, sccl.U8, device=-1, protocol="ll")
    os.environ["SCCL_LL_PARITY"] = "0"
    try:
        b = sccl.Plan(js, 1, 2, 4096, sccl.U8, device=-1, protocol="ll")
    finally:
        os.environ.pop("SCCL_LL_PARITY")
    assert a.info()["region_bytes"] == b.info()["region_bytes"]
    blobs = [a.export_handles(), b.export_handles()]
    with pytest.raises(sccl.InvalidArgumentError, match="LL slot protocol"):
        a.bind_peers(blobs)
