"""Schedules produced by the SMT synthesizer (tools/make_synth_schedules.py,
committed as files: models are not unique) run through the
host verifier, the oracle, and the lowering interpreter."""
import glob
import json
import os
import shutil

import numpy as np
import pytest

import oracle as O
from paper_2008_08708_b200 import sccl

FILES = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "schedules", "*.json")))
NAMES = [os.path.basename(f)[:-5] for f in FILES]


def _load(name):
    return open(os.path.join(os.path.dirname(__file__), "golden", "schedules", name + ".json")).read().strip()


def test_files_present():
    assert len(FILES) >= 9


@pytest.mark.parametrize("name", NAMES)
def test_canonical_and_verified(name):
    js = _load(name)
    assert sccl.canonicalize(js) == js
    assert sccl.verify(js) == []
    assert O.verify(json.loads(js)) == []


def test_table4_allreduce_tuples():
    """SPEC.md:360 / Table 4: DGX-1 AG (1,2,2) -> AR (8,4,4); (2,2,3) -> (16,4,6)."""
    a = json.loads(_load("ar_from_dgx1_1_2_2"))
    b = json.loads(_load("ar_from_dgx1_2_2_3"))
    assert (a["C"], a["S"], a["R"]) == (8, 4, 4)
    assert (b["C"], b["S"], b["R"]) == (16, 4, 6)
    c = json.loads(_load("ar_from_dgx1_6_3_7"))  # the SPEC's own row (acceptance :641)
    assert (c["C"], c["S"], c["R"]) == (48, 6, 14)
    g = json.loads(_load("ag_dgx1_6_3_7"))  # Table 4 (6,3,7): bandwidth-optimal, R/C = 7/6 = b_l
    assert (g["C"], g["S"], g["R"]) == (6, 3, 7) and sum(g["rounds"]) == 7


@pytest.mark.skipif(shutil.which(os.environ.get("SCCL_SOLVER", "z3")) is None, reason="no SMT solver")
def test_symmetric_encoding_small():
    """The symmetry-reduced encoding (DGX-1 automorphism group, order 4,
    acting freely) finds verifier-clean schedules; images of the base
    chunks' routes fill in the rest."""
    from paper_2008_08708_b200 import synth
    grp = synth.automorphisms("dgx1")
    assert len(grp) == 4 and all(g[n] != n for g in grp[1:] for n in range(8))
    st, js, _ = synth.synthesize_symmetric("allgather", "dgx1", 1, 2, 2, timeout=60)
    assert st == "sat" and sccl.verify(js) == []
    d = json.loads(js)
    assert len(d["sends"]) == 56  # exactly once: 8 chunks x 7 receivers


@pytest.mark.parametrize("name", NAMES)
@pytest.mark.parametrize("protocol", ["ll", "simple"])
def test_interpreter_on_synthesized(name, protocol):
    js = _load(name)
    d = json.loads(js)
    kind = d["collective"]
    dt = O.I32 if kind == "allreduce" else O.U8
    nb = 8 * 1000
    ins = O.seeded_inputs(kind, d["P"], nb, dt, 13)
    ref = O.execute(d, ins, nb, dt)
    p = sccl.LoopbackPlan(js, nb, dt, device=-1, protocol=protocol, tile_bytes=256 if protocol == "simple" else 0)
    outs = [np.zeros_like(r) for r in ref]
    p.interpret_on_cpu(ins, outs)
    for a, b in zip(outs, ref):
        assert np.array_equal(a, b)
    if kind == "allreduce":  # exact integer sums (acceptance :641)
        want = np.sum([x.view(np.int32).astype(np.int64) for x in ins], axis=0).astype(np.int32)
        assert all(np.array_equal(o.view(np.int32), want) for o in ref)


@pytest.mark.skipif(shutil.which(os.environ.get("SCCL_SOLVER", "z3")) is None, reason="no SMT solver")
def test_synth_small_instances():
    """Encoding C1-C6 + solver driver: ring(4) needs 2
    steps (diameter); (1,2,2) on DGX-1 is SAT (Table 4 row 1)."""
    from paper_2008_08708_b200 import synth
    assert synth.synthesize("allgather", "ring:4", 1, 1, 1)[0] == "unsat"
    st, js, _ = synth.synthesize("allgather", "ring:4", 1, 2, 2)
    assert st == "sat" and sccl.verify(js) == []
    st, js, _ = synth.synthesize("allgather", "dgx1", 1, 2, 2)
    assert st == "sat" and json.loads(js)["S"] == 2
    st, js, _ = synth.synthesize("broadcast", "ring:4", 2, 3, 3, root=0)
    assert st == "sat" and sccl.verify(js) == []


PARETO = sorted(glob.glob(os.path.join(os.path.dirname(os.path.dirname(__file__)), "paper_2008_08708_b200", "frontiers", "ag_*.json")))


def test_pareto_index_matches_paper():
    """Table 5: ring(8) k=0 frontier starts at (1,4,4);
    k=3 reaches (2,4,7), both latency- and bandwidth-optimal."""
    idx = json.load(open(os.path.join(os.path.dirname(os.path.dirname(__file__)), "paper_2008_08708_b200", "frontiers", "index.json")))
    r8 = {(e["k"], e["C"], e["S"], e["R"]) for e in idx if e["topology"] == "ring:8"}
    assert (0, 1, 4, 4) in r8 and (3, 2, 4, 7) in r8
    assert all(e["bandwidth_optimal"] for e in idx if e["topology"].startswith("full"))


@pytest.mark.parametrize("path", PARETO, ids=[os.path.basename(p)[:-5] for p in PARETO])
def test_pareto_files_verified_and_executable(path):
    js = open(path).read().strip()
    assert sccl.verify(js) == []
    d = json.loads(js)
    ar = sccl.compose_allreduce(sccl.invert(js), js)
    for sched, dt in ((js, O.U8), (ar, O.BF16)):
        dd = json.loads(sched)
        nb = 8 * 300
        ins = O.seeded_inputs(dd["collective"], d["P"], nb, dt, 4)
        ref = O.execute(dd, ins, nb, dt)
        p = sccl.LoopbackPlan(sched, nb, dt, device=-1)
        outs = [np.zeros_like(r) for r in ref]
        p.interpret_on_cpu(ins, outs)
        assert all(np.array_equal(a, b) for a, b in zip(outs, ref))


@pytest.mark.skipif(shutil.which(os.environ.get("SCCL_SOLVER", "z3")) is None, reason="no SMT solver")
def test_pareto_synthesize_small():
    from paper_2008_08708_b200 import synth
    assert synth.diameter("ring:8") == 4 and synth.diameter("dgx1") == 2
    from fractions import Fraction
    assert synth.bandwidth_lower_bound("allgather", "dgx1") == Fraction(7, 6)  # PAPER §2.4
    fr = synth.pareto_synthesize("allgather", "ring:4", 1, max_steps=4, timeout=60)
    assert [(e["C"], e["S"], e["R"]) for e in fr] == [(2, 2, 3)]


@pytest.mark.skipif(shutil.which(os.environ.get("SCCL_SOLVER", "z3")) is None, reason="no SMT solver")
@pytest.mark.timeout(120)
def test_pareto_rooted_kinds_terminate():
    """Gather concentrates the receipts on the root's ingress, scatter the
    sends on its egress: the bandwidth bound is positive, so Algorithm 1's
    (R, C) scan ends (it looped forever with a zero bound)."""
    from fractions import Fraction
    from paper_2008_08708_b200 import synth
    assert synth.bandwidth_lower_bound("gather", "ring:4") == Fraction(3, 2)
    assert synth.bandwidth_lower_bound("scatter", "full:8") == Fraction(1)
    assert synth.bandwidth_lower_bound("broadcast", "full:8") == Fraction(1, 7)
    fr = synth.pareto_synthesize("gather", "ring:4", 0, max_steps=3, timeout=60)
    assert [(e["C"], e["S"], e["R"]) for e in fr] == [(1, 2, 2), (2, 3, 3)]
    assert fr[-1]["bandwidth_optimal"]
    fr = synth.pareto_synthesize("scatter", "full:4", 0, max_steps=3, timeout=60)
    assert [(e["C"], e["S"], e["R"]) for e in fr] == [(1, 1, 1)]
