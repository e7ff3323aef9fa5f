"""Lowering checked on CPU: the per-rank channel program, run by the test-only
CPU interpreter (include/sccl_debug.h; atomics stand in for the flags),
must reproduce the oracle bit for bit -- the same program the GPU kernel
executes."""
import json

import numpy as np
import pytest

import oracle as O
from paper_2008_08708_b200 import sccl
from paper_2008_08708_b200 import schedules as S


def _cases():
    ag8 = S.hamiltonian_allgather(8)
    return {
        "b1": S.to_json(S.recursive_doubling_ring4()), "b2": S.to_json(S.ring4_s2r2()),
        "b3": S.to_json(S.dgx1_allgather_122()), "b4": S.to_json(S.one_shot_allgather(8)),
        "b5": S.to_json(S.direct_alltoall(8)), "b7": S.to_json(S.ring_allgather(8)),
        "b8": S.to_json(S.bidir_ring_allgather(8)), "ham8": S.to_json(ag8),
        "rs_b4": S.reducescatter_from(S.one_shot_allgather(8)), "rs_ring": S.reducescatter_from(S.ring_allgather(8)),
        "ar_b4": S.allreduce_from(S.one_shot_allgather(8)), "ar_ring": S.allreduce_from(S.ring_allgather(8)),
        "ar_ham": S.allreduce_from(ag8), "ar_b1": S.allreduce_from(S.recursive_doubling_ring4()),
        "ar_b3": S.allreduce_from(S.dgx1_allgather_122()), "bcast": S.to_json(S.one_shot_broadcast(4, 3, 1)),
        "chain": S.to_json(S.pipelined_chain_broadcast(5, 4, 2)),
        "reduce": S.reduce_from(S.pipelined_chain_broadcast(5, 4, 2)),
        "gather": S.to_json(S.direct_gather(4, 2)), "scatter": S.to_json(S.direct_scatter(4, 1)),
        "a2a_k2": S.to_json(S.direct_alltoall(4, 8)),
    }


CASES = _cases()


def run_interp(js, nbytes, dtype, nch, tile, seed=7, mode="random"):
    d = json.loads(js)
    ins = O.seeded_inputs(d["collective"], d["P"], nbytes, dtype, seed, mode)
    ref = O.execute(d, ins, nbytes, dtype)
    plan = sccl.LoopbackPlan(js, nbytes, dtype, device=-1, nchannels=nch, tile_bytes=tile)
    outs = [np.zeros_like(r) for r in ref]
    plan.interpret_on_cpu(ins, outs)
    for r, (a, b) in enumerate(zip(outs, ref)):
        assert np.array_equal(a, b), f"rank {r}"


@pytest.mark.parametrize("name", sorted(CASES))
@pytest.mark.parametrize("nbytes", [0, 16, 1000, 4096 + 48])
def test_interpreter_matches_oracle(name, nbytes):
    js = CASES[name]
    kind = json.loads(js)["collective"]
    dts = [O.U8] if kind not in ("reduce", "reducescatter", "allreduce") else [O.U8, O.I32, O.F32, O.BF16, O.F16]
    for dt in dts:
        if nbytes % O.ESIZE[dt] or (kind == "alltoall" and nbytes % (json.loads(js)["P"] * O.ESIZE[dt])):
            continue
        run_interp(js, nbytes, dt, nch=2, tile=256)


@pytest.mark.parametrize("name", ["ar_b4", "ar_ring", "ar_ham", "rs_ring", "reduce"])
@pytest.mark.parametrize("dt", [O.F32, O.BF16, O.F16])
def test_special_values_all_restatements(name, dt):
    """Uniformly random bit patterns (NaN, inf, subnormals, overflow): the
    C oracle, the pure-Python oracle and the host interpreter agree bit for
    bit (canonical NaN rule of DESIGN.md section 2)."""
    js = CASES[name]
    d = json.loads(js)
    ins = O.seeded_inputs(d["collective"], d["P"], 4096, dt, 11, "bits")
    a, b = O.execute(d, ins, 4096, dt), O.execute_py(d, ins, 4096, dt)
    assert all(np.array_equal(x, y) for x, y in zip(a, b))
    run_interp(js, 4096, dt, nch=2, tile=256, seed=11, mode="bits")


@pytest.mark.parametrize("nch,tile", [(1, 256), (3, 272), (5, 4096)])
def test_interpreter_channels_tiles(nch, tile):
    for name in ("ham8", "ar_ham", "rs_ring", "a2a_k2"):
        js = CASES[name]
        kind = json.loads(js)["collective"]
        run_interp(js, 3000 + 200, O.BF16 if kind in ("allreduce", "reducescatter") else O.U8, nch, tile)


def test_program_structure_one_shot_allgather():
    """B4 lowers to exactly one fused op per rank: read the input chunk once,
    write the own output slot and the 7 peers (PAPER.md:724 single fused
    kernel, push model PAPER.md:720), plus the end-of-program wait."""
    plan = sccl.LoopbackPlan(CASES["b4"], 1 << 20, sccl.U8, device=-1, protocol="simple")
    prog = plan.info()["program"]
    for r, rk in enumerate(prog["ranks"]):
        kinds = [op["kind"] for op in rk["ops"]]
        assert kinds == ["copy", "wait"]
        assert len(rk["ops"][0]["outs"]) == 8
        assert len(rk["ops"][1]["ins"]) == 7


def test_program_structure_fused_allreduce():
    """(8,2,2) push lowering: per rank 7 pushes into peers' receipt slots,
    then one fused receive-reduce-broadcast op (8 inputs, 8 outputs)."""
    plan = sccl.LoopbackPlan(CASES["ar_b4"], 1 << 20, sccl.BF16, device=-1, protocol="simple", pull="off")
    assert plan.info()["pull"] == 0
    for rk in plan.info()["program"]["ranks"]:
        red = [op for op in rk["ops"] if op["kind"] == "reduce"]
        assert len(red) == 1 and len(red[0]["ins"]) == 8 and len(red[0]["outs"]) == 8
        assert sum(op["kind"] == "copy" for op in rk["ops"]) == 7


def test_program_structure_pull_allreduce():
    """(8,2,2) pull lowering (loopback default): the reduce-scatter sends of
    untouched inputs become in-place reads of the peers' SEND buffers by the
    home rank's reduce -- no copies, no receipt slots, no scratch; inputs in
    the schedule's order (own value first, then sources ascending)."""
    plan = sccl.LoopbackPlan(CASES["ar_b4"], 1 << 20, sccl.BF16, device=-1, protocol="simple")
    info = plan.info()
    assert info["pull"] == 1 and info["program"]["scratch_bytes"] == 0
    for r, rk in enumerate(info["program"]["ranks"]):
        assert [op["kind"] for op in rk["ops"]] == ["reduce", "wait"]
        red = rk["ops"][0]
        assert [i[0] for i in red["ins"]] == [r] + [s for s in range(8) if s != r]
        assert all(i[1] == "send" and i[3] == -1 for i in red["ins"])
        assert len(red["outs"]) == 8


def test_pull_first_hop_of_chains():
    """Reduction chains pull only their first hop (the sender's untouched
    input); later hops read partial sums, which still travel as receipts."""
    push = sccl.LoopbackPlan(CASES["ar_ring"], 1 << 16, sccl.F32, device=-1, protocol="simple", pull="off").info()
    pull = sccl.LoopbackPlan(CASES["ar_ring"], 1 << 16, sccl.F32, device=-1, protocol="simple").info()
    ncopy = lambda info: sum(op["kind"] == "copy" for rk in info["program"]["ranks"] for op in rk["ops"])
    remote = [i for rk_i, rk in enumerate(pull["program"]["ranks"]) for op in rk["ops"] if op["kind"] == "reduce"
              for i in op["ins"] if i[0] != rk_i]
    assert remote and all(i[1] == "send" for i in remote)
    assert ncopy(pull) == ncopy(push) - 8  # one first-hop send per chunk


def test_pull_rejected_for_multiprocess():
    with pytest.raises(sccl.InvalidArgumentError):
        sccl.Plan(CASES["ar_b4"], 0, 8, 1 << 16, sccl.BF16, device=-1, pull="on")


def test_dead_partial_store_elided():
    """Ring allreduce: a non-home partial sum is forwarded inside the fused
    op and never stored locally (the allgather phase overwrites it)."""
    plan = sccl.LoopbackPlan(CASES["ar_ring"], 1 << 16, sccl.F32, device=-1)
    for r, rk in enumerate(plan.info()["program"]["ranks"]):
        for op in rk["ops"]:
            if op["kind"] == "reduce" and op["chunk"] % 8 != r:
                assert all(o[0] != r for o in op["outs"]), op


def test_fingerprint_stable_across_ranks():
    a = sccl.Plan(CASES["ham8"], 0, 8, 1 << 20, sccl.U8, device=-1)
    b = sccl.Plan(CASES["ham8"], 5, 8, 1 << 20, sccl.U8, device=-1)
    assert a.info()["program"]["fingerprint"] == b.info()["program"]["fingerprint"]
    c = sccl.Plan(CASES["ham8"], 5, 8, 1 << 21, sccl.U8, device=-1)
    assert c.info()["program"]["fingerprint"] != a.info()["program"]["fingerprint"]


@pytest.mark.parametrize("kc,kb", [(3, 1), (2, 3), (56, 1), (7, 2)])
def test_interpreter_chunk_groups(kc, kb):
    """channel j = (chunk group j % kc, byte part j / kc): independent chunks
    on different CTAs, each chunk's ops still in program order."""
    plan_js = [CASES["ham8"], CASES["ar_ham"], CASES["b5"], CASES["reduce"]]
    for js in plan_js:
        d = json.loads(js)
        kind = d["collective"]
        dt = O.BF16 if kind in ("allreduce", "reducescatter", "reduce") else O.U8
        nbytes = 8 * 600
        ins = O.seeded_inputs(kind, d["P"], nbytes, dt, 3)
        ref = O.execute(d, ins, nbytes, dt)
        plan = sccl.LoopbackPlan(js, nbytes, dt, device=-1, nchannels=kb, chunk_groups=kc, tile_bytes=256)
        info = plan.info()
        assert info["chunk_groups"] == kc and info["byte_parts"] == kb
        outs = [np.zeros_like(r) for r in ref]
        plan.interpret_on_cpu(ins, outs)
        assert all(np.array_equal(a, b) for a, b in zip(outs, ref))


def test_auto_channel_policy():
    """Small chunks spread over chunk groups (latency); large chunks cut into
    byte parts (bandwidth)."""
    small = sccl.LoopbackPlan(CASES["ham8"], 1024, sccl.U8, device=-1).info()
    assert small["chunk_groups"] > 1 and small["byte_parts"] == 1 and small["storer_warps"] == 3
    large = sccl.LoopbackPlan(CASES["ham8"], 64 << 20, sccl.U8, device=-1).info()
    assert large["byte_parts"] > 1 and large["tile_bytes"] == 32768 and large["nstage"] % 3 == 0
