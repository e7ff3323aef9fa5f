"""Per-size algorithm + protocol selection (SPEC.md:456-509,
PAPER.md:1037): sccl_schedule_select over a candidate set, checked against
the B200 loopback Pareto sweep committed in tests/golden (BASELINE config 5,
measured by tools/pareto_sweep.py)."""
import json
import os

import pytest

from paper_2008_08708_b200 import sccl
from paper_2008_08708_b200 import schedules as S

HERE = os.path.dirname(__file__)
PARETO = os.path.join(os.path.dirname(HERE), "paper_2008_08708_b200", "frontiers")


def frontier_candidates():
    index = json.load(open(os.path.join(PARETO, "index.json")))
    seen, cands = set(), {}
    for e in index:
        key = (e["topology"], e["C"], e["S"], e["R"])
        if key in seen:
            continue
        seen.add(key)
        ag = open(os.path.join(PARETO, e["file"])).read().strip()
        ar = sccl.compose_allreduce(sccl.invert(ag), ag)
        cands.setdefault((e["P"], "allgather"), []).append(((e["topology"], e["C"], e["S"], e["R"]), ag))
        cands.setdefault((e["P"], "allreduce"), []).append(
            ((e["topology"], e["C"] * e["P"], e["S"] * 2, e["R"] * 2), ar))
    return cands


def test_select_api():
    P = 8
    c = [S.to_json(S.hamiltonian_allgather(P)), S.to_json(S.one_shot_allgather(P))]
    i, proto, us = sccl.select(c, 1 << 10)
    assert i in (0, 1) and proto in ("ll", "simple") and us > 0
    # latency-bound: LL; bandwidth-bound: the bulk protocol
    assert sccl.select(c, 1 << 10)[1] == "ll"
    assert sccl.select(c, 1 << 28)[1] == "simple"
    # predicted time grows with size
    assert sccl.select(c, 1 << 28)[2] > sccl.select(c, 1 << 20)[2] > sccl.select(c, 1 << 10)[2]


def test_select_rejects_bad_input():
    P = 8
    with pytest.raises(sccl.InvalidArgumentError):
        sccl.select([], 1024)
    with pytest.raises(sccl.InvalidArgumentError):  # mixed collectives
        sccl.select([S.to_json(S.one_shot_allgather(P)), S.to_json(S.direct_alltoall(P))], 1024)
    with pytest.raises(sccl.InvalidArgumentError):  # mixed P
        sccl.select([S.to_json(S.one_shot_allgather(4)), S.to_json(S.one_shot_allgather(8))], 1024)
    bad = json.loads(S.to_json(S.one_shot_allgather(P)))
    bad["sends"] = bad["sends"][:-1]  # post-condition violated: unverified schedules are rejected
    with pytest.raises(sccl.InvalidArgumentError):
        sccl.select([json.dumps(bad)], 1024)


def test_select_regret_vs_measured_b200_frontier():
    """The model's pick among each committed frontier, per size, against the
    measured B200 times of every frontier member: mean regret <= 10 %."""
    meas = [json.loads(x) for x in open(os.path.join(HERE, "golden", "pareto_measured_b200.jsonl"))
            if '"summary"' not in x]
    regrets = []
    for (P, coll), cl in frontier_candidates().items():
        for sz in sorted({m["bytes_per_rank"] for m in meas}):
            rows = {(m["topology"], m["C"], m["S"], m["R"]): m["us"] for m in meas
                    if m["P"] == P and m["collective"] == coll and m["bytes_per_rank"] == sz}
            i, _, _ = sccl.select([c[1] for c in cl], sz, sccl.U8 if coll == "allgather" else sccl.BF16)
            regrets.append(rows[cl[i][0]] / min(rows.values()) - 1)
    assert len(regrets) == 42
    assert sum(regrets) / len(regrets) <= 0.10, regrets


def test_auto_plan_caches_per_size():
    c = [S.to_json(S.hamiltonian_allgather(8)), S.to_json(S.one_shot_allgather(8))]
    auto = sccl.AutoLoopbackPlan(c, sccl.U8, device=-1, max_plans=2)
    a = auto.plan_for(1024)
    assert auto.plan_for(1024) is a          # cached
    assert a[1] == "ll"
    auto.plan_for(1 << 20)
    auto.plan_for(1 << 24)                   # evicts the oldest (1024)
    assert 1024 not in auto._plans and len(auto._plans) == 2
    auto.close()
