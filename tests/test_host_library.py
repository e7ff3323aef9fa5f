"""C++ host library (through the C-ABI): schedule IR, canonical JSON,
verify / verify_combining, inversion, composition -- checked against the
SPEC examples and the independent oracle restatement."""
import json
import random

import numpy as np
import pytest

import oracle as O
from paper_2008_08708_b200 import sccl
from paper_2008_08708_b200 import schedules as S


def _kinds(v):
    names = {1: "schema", 2: "edge", 3: "unavailable", 4: "bandwidth", 5: "post", 6: "duplicate",
             7: "multiplicity"}
    return {names[x[0]] for x in v}


ALL = {
    "b1": S.recursive_doubling_ring4(), "b2": S.ring4_s2r2(), "b3": S.dgx1_allgather_122(),
    "b4": S.one_shot_allgather(8), "b5": S.direct_alltoall(8), "b7": S.ring_allgather(8),
    "b8": S.bidir_ring_allgather(8), "ham8": S.hamiltonian_allgather(8), "ham5": S.hamiltonian_allgather(5),
    "bc": S.one_shot_broadcast(4, 3, 1), "chain": S.pipelined_chain_broadcast(5, 4, 2),
    "ga": S.direct_gather(4, 2), "sc": S.direct_scatter(4, 1),
}


@pytest.mark.parametrize("name", sorted(ALL))
def test_known_schedules_verify_in_both(name):
    js = S.to_json(ALL[name])
    assert sccl.verify(js) == []
    assert O.verify(json.loads(js)) == []


@pytest.mark.parametrize("name", sorted(ALL))
def test_canonical_roundtrip_byte_identical(name):
    """round trip identity; two serializations identical;
    sends sorted by (step, chunk, src, dst)."""
    js = S.to_json(ALL[name])
    assert sccl.canonicalize(js) == js
    d = json.loads(js)
    shuffled = dict(d)
    sends = list(d["sends"])
    random.Random(1).shuffle(sends)
    shuffled["sends"] = sends
    assert sccl.canonicalize(json.dumps(shuffled, indent=2)) == js
    assert d["sends"] == sorted(d["sends"], key=lambda t: (t[3], t[0], t[1], t[2]))


def test_topology_hash_matches_oracle():
    for name in ("ring:4", "ring:8", "full:8", "dgx1", "amd-z52", "switch:8", "full:2"):
        d = json.loads(S.to_json(S._sched("allgather", name, O.topology_by_name(name)["P"],
                                          O.topology_by_name(name)["P"], 1, [1], [])))
        assert d["topology"]["hash"] == O.topology_hash(O.topology_by_name(name))


def test_schema_errors():
    """step >= S is a schema error; bad hash is rejected."""
    d = json.loads(S.to_json(S.recursive_doubling_ring4()))
    bad = dict(d, sends=d["sends"] + [[0, 0, 1, 2]])
    with pytest.raises(sccl.InvalidArgumentError, match="step >= S"):
        sccl.canonicalize(json.dumps(bad))
    bad = json.loads(json.dumps(d))
    bad["topology"]["hash"] = "0" * 16
    with pytest.raises(sccl.InvalidArgumentError, match="hash mismatch"):
        sccl.canonicalize(json.dumps(bad))
    with pytest.raises(sccl.InvalidArgumentError):
        sccl.canonicalize("{not json")
    bad = dict(d, G=5)
    with pytest.raises(sccl.InvalidArgumentError, match="to_global"):
        sccl.canonicalize(json.dumps(bad))
    bad = dict(d, rounds=[1, 0])
    with pytest.raises(sccl.InvalidArgumentError):
        sccl.canonicalize(json.dumps(bad))


def test_verify_kats_fig2():
    """SPEC.md:406-408."""
    d = json.loads(S.to_json(S.recursive_doubling_ring4()))
    assert sccl.verify(d) == []
    assert "post" in _kinds(sccl.verify(dict(d, sends=d["sends"][1:])))
    shifted = dict(d, sends=[[c, a, b, 0] for c, a, b, _ in d["sends"]])
    assert "bandwidth" in _kinds(sccl.verify(shifted))


def test_invert_involution_and_tuple():
    """invert(invert(s)) = s; AR tuple (P*C,2S,2R)."""
    for ag in (S.recursive_doubling_ring4(), S.dgx1_allgather_122(), S.hamiltonian_allgather(8)):
        js = S.to_json(ag)
        rs = sccl.invert(js)
        assert json.loads(rs)["collective"] == "reducescatter"
        assert sccl.verify(rs) == []
        assert sccl.invert(rs) == js
        ar = json.loads(sccl.compose_allreduce(rs, js))
        d = json.loads(js)
        assert (ar["C"], ar["S"], ar["R"]) == (d["P"] * d["C"], 2 * d["S"], 2 * d["R"])
    # Table 4 rows: DGX-1 AG (1,2,2) -> AR (8,4,4)
    ar = json.loads(S.allreduce_from(S.dgx1_allgather_122()))
    assert (ar["C"], ar["S"], ar["R"]) == (8, 4, 4)
    # {(0,0,1,0)} with S=1 -> {(0,1,0,0)}
    assert json.loads(sccl.invert(S.two_node_send()))["sends"] == [[0, 1, 0, 0]]


def test_composition_rejects_mismatch():
    with pytest.raises(sccl.InvalidArgumentError):
        sccl.compose_allreduce(S.to_json(S.ring_allgather(8)), S.to_json(S.ring_allgather(8)))


def _mutate(d, rng):
    d = json.loads(json.dumps(d))
    sends = d["sends"]
    op = rng.choice(["delete", "dup", "shift", "edge", "swap"])
    i = rng.randrange(len(sends))
    if op == "delete":
        sends.pop(i)
    elif op == "dup":
        c, a, b, s = sends[i]
        sends.append([c, a, b, rng.randrange(d["S"])])
    elif op == "shift":
        sends[i][3] = rng.randrange(d["S"])
    elif op == "edge":
        x = rng.randrange(d["P"])
        if x != sends[i][1]:
            sends[i][2] = x
    else:
        j = rng.randrange(len(sends))
        sends[i][0], sends[j][0] = sends[j][0], sends[i][0]
    return d


def test_mutation_corpus_cpp_equals_oracle():
    """Acceptance SPEC.md:644: 1000 random mutations; the C++ verifier and
    the independent oracle verifier agree on every mutant (same violation
    kinds), combining and non-combining."""
    rng = random.Random(7)
    bases = [json.loads(S.to_json(x)) for x in ALL.values()]
    bases += [json.loads(sccl.invert(S.ring_allgather(8))), json.loads(sccl.invert(S.recursive_doubling_ring4())),
              json.loads(sccl.invert(S.pipelined_chain_broadcast(5, 4, 2)))]
    n = 0
    while n < 1000:
        d = _mutate(rng.choice(bases), rng)
        try:
            cv = sccl.verify(d)
        except sccl.InvalidArgumentError:
            continue  # schema-level (e.g. src == dst) rejected by deserialize
        ov = O.verify(d)
        assert _kinds(cv) == {v[0] for v in ov}, (d, cv, ov)
        assert len(cv) == len(ov)
        n += 1


@pytest.mark.parametrize("name", ["b1", "b3", "ham8"])
def test_unverified_schedule_rejected_by_plan(name):
    """executing an unverified schedule is rejected."""
    d = json.loads(S.to_json(ALL[name]))
    d["sends"] = d["sends"][:-1]
    with pytest.raises(sccl.InvalidArgumentError, match="unverified"):
        sccl.LoopbackPlan(d, 4096, sccl.U8, device=-1)
