"""LL protocol lowering (flag-in-data receipts) checked on CPU by the
test-only interpreter against the oracle; zero-length and ragged chunks."""
import json

import numpy as np
import pytest

import oracle as O
from paper_2008_08708_b200 import sccl
from paper_2008_08708_b200 import schedules as S

CASES = {
    "ham8": S.to_json(S.hamiltonian_allgather(8)), "ar_ham": S.allreduce_from(S.hamiltonian_allgather(8)),
    "a2a": S.to_json(S.direct_alltoall(8)), "reduce": S.reduce_from(S.pipelined_chain_broadcast(5, 4, 2)),
    "ar_ring": S.allreduce_from(S.ring_allgather(8)), "gather": S.to_json(S.direct_gather(4, 2)),
    "b3": S.to_json(S.dgx1_allgather_122()), "ar_822": S.allreduce_from(S.one_shot_allgather(8)),
}


@pytest.mark.parametrize("name", sorted(CASES))
@pytest.mark.parametrize("nb", [0, 8, 24, 1000, 4096 + 48, 20000])
@pytest.mark.parametrize("kc,kb", [(0, 0), (3, 2)])
@pytest.mark.parametrize("protocol", ["ll", "simple"])
def test_protocols_match_oracle(name, nb, kc, kb, protocol):
    js = CASES[name]
    d = json.loads(js)
    kind = d["collective"]
    dts = [O.U8] if kind not in ("allreduce", "reduce", "reducescatter") else [O.U8, O.I32, O.F32, O.BF16, O.F16]
    for dt in dts:
        if nb % O.ESIZE[dt] or (kind == "alltoall" and nb % (8 * O.ESIZE[dt])):
            continue
        ins = O.seeded_inputs(kind, d["P"], nb, dt, 5)
        ref = O.execute(d, ins, nb, dt)
        p = sccl.LoopbackPlan(js, nb, dt, device=-1, protocol=protocol, nchannels=kb, chunk_groups=kc,
                              tile_bytes=256 if protocol == "simple" else 0)
        assert p.info()["protocol"] == protocol
        outs = [np.zeros_like(r) for r in ref]
        p.interpret_on_cpu(ins, outs)
        for r, (a, b) in enumerate(zip(outs, ref)):
            assert np.array_equal(a, b), (name, dt, nb, r)


def test_auto_protocol_by_size():
    js = CASES["ham8"]
    assert sccl.LoopbackPlan(js, 4096, sccl.U8, device=-1).info()["protocol"] == "ll"
    assert sccl.LoopbackPlan(js, 64 << 20, sccl.U8, device=-1).info()["protocol"] == "simple"


def test_ll_program_has_no_end_waits():
    """LL: every receipt is consumed by an unpacking/forwarding op (the
    local copy of a post entry is fused with the forward of the same
    receipt), so no end-of-program counter waits remain."""
    p = sccl.LoopbackPlan(CASES["ham8"], 4096, sccl.U8, device=-1, protocol="ll")
    for rk in p.info()["program"]["ranks"]:
        assert all(op["kind"] != "wait" for op in rk["ops"])
