"""GPU parity: the sm_100a executor (through the C-ABI) against the CPU oracle.

Bit-exact for every collective and element type: copies are bitwise, and
reductions follow the fixed order the oracle defines (DESIGN.md "Reduction
order"); no tolerance is needed or used.  Loopback mode runs every rank of
the schedule on cuda:0 (one launch, P x nchannels CTAs).
"""
import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle as O  # noqa: E402
from paper_2008_08708_b200 import sccl  # noqa: E402
from paper_2008_08708_b200 import schedules as S  # noqa: E402

pytestmark = pytest.mark.gpu

DEV = "cuda:0"


def _schedules():
    ag8 = S.hamiltonian_allgather(8)
    return {
        "ag_b1_recdbl": S.to_json(S.recursive_doubling_ring4()),
        "ag_b2_ring4": S.to_json(S.ring4_s2r2()),
        "ag_b3_dgx1": S.to_json(S.dgx1_allgather_122()),
        "ag_b4_oneshot8": S.to_json(S.one_shot_allgather(8)),
        "ag_b7_ring8": S.to_json(S.ring_allgather(8)),
        "ag_b8_bidir8": S.to_json(S.bidir_ring_allgather(8)),
        "ag_777": S.to_json(ag8),
        "a2a_b5": S.to_json(S.direct_alltoall(8)),
        "a2a_k2": S.to_json(S.direct_alltoall(4, 8)),
        "bcast": S.to_json(S.one_shot_broadcast(4, 3, 1)),
        "bcast_chain": S.to_json(S.pipelined_chain_broadcast(5, 4, 2)),
        "gather": S.to_json(S.direct_gather(4, 2)),
        "scatter": S.to_json(S.direct_scatter(4, 1)),
        "rs_oneshot8": S.reducescatter_from(S.one_shot_allgather(8)),
        "rs_ring8": S.reducescatter_from(S.ring_allgather(8)),
        "reduce_chain": S.reduce_from(S.pipelined_chain_broadcast(5, 4, 2)),
        "ar_822": S.allreduce_from(S.one_shot_allgather(8)),
        "ar_ring": S.allreduce_from(S.ring_allgather(8)),
        "ar_56_14_14": S.allreduce_from(ag8),
        "ar_dgx1": S.allreduce_from(S.dgx1_allgather_122()),
        "ar_recdbl": S.allreduce_from(S.recursive_doubling_ring4()),
    }


SCHED = _schedules()


def run_gpu(js, nbytes, dtype, seed=3, mode="random", nch=0, tile=0, repeats=1, protocol="auto", kc=0,
            pull="auto"):
    """Launch the plan on sentinel-filled (0xEE) outputs; every byte the
    collective defines must equal the oracle's, every other byte must still
    be the sentinel (a kernel that clobbers a non-root or out-of-post byte
    fails)."""
    d = json.loads(js)
    kind, P = d["collective"], d["P"]
    plan = sccl.LoopbackPlan(js, nbytes, dtype, device=0, nchannels=nch, tile_bytes=tile, protocol=protocol,
                             chunk_groups=kc, pull=pull)
    try:
        for it in range(repeats):
            ins = O.seeded_inputs(kind, P, nbytes, dtype, seed + it, mode)
            ref = O.execute(d, ins, nbytes, dtype)
            send = [torch.from_numpy(x).to(DEV) for x in ins]
            recv = [torch.full((max(r.size, 1),), 0xEE, dtype=torch.uint8, device=DEV) for r in ref]
            plan.launch(send, recv)
            torch.cuda.synchronize()
            plan.check()
            for r, (a, b) in enumerate(zip(recv, ref)):
                got = a.cpu().numpy()[:b.size]
                mask = _covered(d, nbytes, r, b.size)
                assert np.array_equal(got[mask], b[mask]), f"{kind} rank {r} iter {it} differs"
                assert np.all(got[~mask] == 0xEE), f"{kind} rank {r} iter {it}: bytes outside the post-condition written"
    finally:
        plan.close()


def _covered(d, nbytes, rank, size):
    """bytes of rank's output that the collective defines (rooted
    collectives leave non-root outputs untouched)."""
    kind = d["collective"]
    P = d["P"]
    phases = d["phases"] if "phases" in d else [d]
    G = phases[-1]["G"]
    _, post = O.pre_post(phases[-1]["collective"], G, P, d.get("root", 0) or 0)
    C = G // P if kind not in ("broadcast", "reduce") else G
    geo = O.chunk_geometry(kind, P, C, nbytes, G)
    m = np.zeros(size, bool)
    for c in range(G):
        if post[c, rank]:
            m[geo[c][2]:geo[c][2] + geo[c][0]] = True
    return m


@pytest.mark.parametrize("name", sorted(SCHED))
@pytest.mark.parametrize("nbytes", [0, 16, 1040, 65536 + 32, 1 << 20])
def test_parity_u8_and_float(name, nbytes):
    js = SCHED[name]
    kind = json.loads(js)["collective"]
    dts = [O.U8] if kind not in ("reduce", "reducescatter", "allreduce") else [O.I32, O.F32, O.BF16, O.F16, O.U8]
    for dt in dts:
        if nbytes % O.ESIZE[dt]:
            continue
        if kind == "alltoall" and nbytes % (json.loads(js)["P"] * O.ESIZE[dt]):
            continue
        run_gpu(js, nbytes, dt)


@pytest.mark.parametrize("pull", ["on", "off"])
@pytest.mark.parametrize("protocol", ["simple", "ll"])
@pytest.mark.parametrize("name", ["rs_oneshot8", "rs_ring8", "reduce_chain", "ar_822", "ar_ring", "ar_56_14_14",
                                  "ar_dgx1", "ar_recdbl"])
def test_pull_and_push_lowering(name, protocol, pull):
    """Combining sends of untouched inputs read in place by the receiver
    (pull, the loopback default) or pushed into receipt slots: the same
    reduction order and operands, so the same bits either way."""
    for nbytes, dt in ((1040, O.F32), (65536 + 32, O.BF16), (1 << 20, O.F16), (3 << 20, O.BF16)):
        if protocol == "ll" and nbytes > (1 << 20):
            continue
        run_gpu(SCHED[name], nbytes, dt, protocol=protocol, pull=pull, repeats=2)


@pytest.mark.parametrize("name", ["ar_822", "ar_56_14_14", "ar_ring", "ar_dgx1"])
@pytest.mark.parametrize("protocol", ["simple", "ll"])
def test_inplace_allreduce_pull(name, protocol):
    """In place (recvbuf == sendbuf) under the pull lowering: a peer's input
    is read in place only if its owner never reduces into that chunk slot,
    so no read races the owner's write."""
    js = SCHED[name]
    d = json.loads(js)
    nbytes = (1 << 20) if protocol == "simple" else (64 << 10)
    for it in range(2):
        ins = O.seeded_inputs("allreduce", 8, nbytes, O.BF16, 40 + it)
        ref = O.execute(d, ins, nbytes, O.BF16)
        plan = sccl.LoopbackPlan(js, nbytes, O.BF16, device=0, protocol=protocol)
        bufs = [torch.from_numpy(x).to(DEV) for x in ins]
        plan.launch(bufs, bufs)
        torch.cuda.synchronize()
        plan.check()
        for a, b in zip(bufs, ref):
            assert np.array_equal(a.cpu().numpy(), b)
        plan.close()


@pytest.mark.parametrize("nch,tile", [(1, 256), (3, 4096), (7, 32768), (0, 0)])
@pytest.mark.parametrize("name", ["ag_777", "ag_b7_ring8", "ar_56_14_14", "ar_ring", "rs_ring8", "a2a_b5"])
def test_channels_and_tiles(name, nch, tile):
    js = SCHED[name]
    kind = json.loads(js)["collective"]
    dt = O.BF16 if kind in ("allreduce", "reducescatter") else O.U8
    run_gpu(js, 3 * 65536 + 1024, dt, nch=nch, tile=tile)


@pytest.mark.parametrize("dt", [O.BF16, O.F16, O.F32])
@pytest.mark.parametrize("name,nbytes", [("ar_ring", 1 << 20), ("ar_56_14_14", 1 << 20), ("ar_822", 1 << 20),
                                         ("rs_ring8", 1 << 18)])
@pytest.mark.parametrize("protocol", ["simple", "ll"])
def test_reduce_special_values(name, nbytes, dt, protocol):
    """Float reductions over uniformly random bit patterns (subnormals,
    infinities, NaNs, overflow to infinity): bit-exact with the oracle's
    widen / add in order / round once / canonical NaN rule, for 2-input
    chain reduces and wide one-shot reduces."""
    run_gpu(SCHED[name], nbytes, dt, mode="bits", protocol=protocol, repeats=2)


@pytest.mark.parametrize("name,nbytes,dt", [
    ("ag_777", 256 << 10, O.U8),          # LL chain: one 37 KiB chunk per CTA
    ("ar_56_14_14", 2 << 20, O.BF16),     # LL chain at its largest chunk (37 KiB)
    ("ar_822", 128 << 10, O.BF16),        # LL: chunks split to 2 KiB parts when groups run out
    ("ar_822", 1 << 20, O.BF16),          # bulk: wide reduce with 16 KiB tiles
    ("ag_b4_oneshot8", 256 << 10, O.U8),  # bulk: one-shot copy with 16 KiB tiles
    ("a2a_b5", 4 << 20, O.U8),            # balanced chunk-group map (chunk % kc is lopsided)
    ("a2a_b5", 2 << 20, O.U8),
])
def test_plan_policy_cases(name, nbytes, dt):
    """The size-dependent channel / tile rules, at the sizes that trigger
    them, under the automatic protocol choice: bit-exact, twice in a row."""
    run_gpu(SCHED[name], nbytes, dt, repeats=2)


def test_back_to_back_launches_advance_epochs():
    run_gpu(SCHED["ar_56_14_14"], 1 << 18, O.F32, repeats=5)
    run_gpu(SCHED["ag_777"], 1 << 18, O.U8, repeats=5, tile=4096)


def test_inplace_allreduce():
    js = SCHED["ar_56_14_14"]
    d = json.loads(js)
    nbytes = 1 << 20
    ins = O.seeded_inputs("allreduce", 8, nbytes, O.F32, 5)
    ref = O.execute(d, ins, nbytes, O.F32)
    plan = sccl.LoopbackPlan(js, nbytes, O.F32, device=0)
    bufs = [torch.from_numpy(x).to(DEV) for x in ins]
    plan.launch(bufs, bufs)
    torch.cuda.synchronize()
    for a, b in zip(bufs, ref):
        assert np.array_equal(a.cpu().numpy(), b)


def test_cuda_graph_replay():
    js = SCHED["ar_822"]
    d = json.loads(js)
    nbytes = 1 << 16
    plan = sccl.LoopbackPlan(js, nbytes, O.BF16, device=0)
    send = [torch.zeros(nbytes, dtype=torch.uint8, device=DEV) for _ in range(8)]
    recv = [torch.zeros(nbytes, dtype=torch.uint8, device=DEV) for _ in range(8)]
    s = torch.cuda.Stream()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        plan.launch(send, recv, stream=s)
    for it in range(3):
        ins = O.seeded_inputs("allreduce", 8, nbytes, O.BF16, 100 + it)
        for t, x in zip(send, ins):
            t.copy_(torch.from_numpy(x))
        g.replay()
        torch.cuda.synchronize()
        ref = O.execute(d, ins, nbytes, O.BF16)
        for a, b in zip(recv, ref):
            assert np.array_equal(a.cpu().numpy(), b), f"graph replay {it}"


@pytest.mark.parametrize("name", ["ag_777", "ag_b4_oneshot8"])
def test_allgather_large_property(name):
    """64 MiB per rank: output of every rank == concatenation of the inputs."""
    js = SCHED[name]
    m = 64 << 20
    plan = sccl.LoopbackPlan(js, m, O.U8, device=0)
    g = torch.Generator(device=DEV)
    g.manual_seed(0)
    send = [torch.randint(0, 256, (m,), dtype=torch.uint8, device=DEV, generator=g) for _ in range(8)]
    recv = [torch.empty(8 * m, dtype=torch.uint8, device=DEV) for _ in range(8)]
    plan.launch(send, recv)
    torch.cuda.synchronize()
    want = torch.cat(send)
    for r in recv:
        assert torch.equal(r, want)


@pytest.mark.parametrize("dt", [O.F32, O.BF16, O.I32])
def test_allreduce_large_exact_sum(dt):
    """64 MiB: integer-valued inputs in [-16,16] make the sum exact in any
    order, so every rank must equal the torch sum bit for bit."""
    js = SCHED["ar_56_14_14"]
    M = 64 << 20
    tdt = {O.F32: torch.float32, O.BF16: torch.bfloat16, O.I32: torch.int32}[dt]
    plan = sccl.LoopbackPlan(js, M, dt, device=0)
    g = torch.Generator(device=DEV)
    g.manual_seed(1)
    n = M // O.ESIZE[dt]
    xs = [torch.randint(-16, 17, (n,), device=DEV, generator=g).to(tdt) for _ in range(8)]
    send = [x.view(torch.uint8) for x in xs]
    recv = [torch.empty(M, dtype=torch.uint8, device=DEV) for _ in range(8)]
    plan.launch(send, recv)
    torch.cuda.synchronize()
    want = torch.stack([x.to(torch.float64) for x in xs]).sum(0).to(tdt).view(torch.uint8)
    for r in recv:
        assert torch.equal(r, want)


@pytest.mark.parametrize("selfpub", ["0", "1"])
@pytest.mark.parametrize("name,nbytes", [("ag_777", 4 << 20), ("ar_56_14_14", 4 << 20), ("ag_b7_ring8", 1 << 20),
                                         ("a2a_b5", 8 << 20), ("ar_822", 1 << 20)])
def test_counter_release_modes(monkeypatch, selfpub, name, nbytes):
    """Both counter-release modes of the bulk protocol (storer warps publish
    their own tiles / the windowed signaler warp), forced, bit-exact."""
    monkeypatch.setenv("SCCL_SELFPUB", selfpub)
    js = SCHED[name]
    dt = O.BF16 if name.startswith("ar") else O.U8
    run_gpu(js, nbytes, dt, protocol="simple", repeats=2)


@pytest.mark.parametrize("P", [2, 3, 5, 6, 16])
@pytest.mark.parametrize("protocol", ["ll", "simple"])
def test_rank_counts(P, protocol):
    """Odd, non-power-of-two and the maximum (16, the kernel's pointer
    table) rank counts: one-shot and ring allgathers, the ring allreduce,
    the direct alltoall, at an unaligned size."""
    nb = 8 * 1000 + 48
    cases = [(S.to_json(S.one_shot_allgather(P)), O.U8), (S.to_json(S.ring_allgather(P)), O.U8),
             (S.allreduce_from(S.ring_allgather(P)), O.BF16), (S.to_json(S.direct_alltoall(P)), O.U8)]
    if P <= 8 and P not in (4, 6):  # K_4* and K_6* have no Hamiltonian decomposition
        cases.append((S.to_json(S.hamiltonian_allgather(P)), O.U8))
    for js, dt in cases:
        run_gpu(js, nb if json.loads(js)["collective"] != "alltoall" else P * 1024, dt, protocol=protocol)


def test_concurrent_distinct_plans():
    """Three loopback plans (both protocols) with disjoint flags/scratch on
    three streams at once (grids that fit together), each bit-exact."""
    cases = [(SCHED["ag_b7_ring8"], 4096, O.U8, 5, "ll"), (SCHED["ar_822"], 1 << 16, O.BF16, 6, "ll"),
             (SCHED["ag_777"], 1 << 20, O.U8, 7, "simple")]
    plans = [sccl.LoopbackPlan(js, nb, dt, device=0, nchannels=2, chunk_groups=1, protocol=pr)
             for js, nb, dt, _, pr in cases]
    assert sum(pl.info()["grid"] for pl in plans) <= 148
    outs = []
    for plan, (js, nb, dt, seed, _) in zip(plans, cases):
        d = json.loads(js)
        ins = O.seeded_inputs(d["collective"], d["P"], nb, dt, seed)
        ref = O.execute(d, ins, nb, dt)
        send = [torch.from_numpy(x).to(DEV) for x in ins]
        recv = [torch.zeros(r.size, dtype=torch.uint8, device=DEV) for r in ref]
        outs.append((plan, send, recv, ref))
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in outs]
    for _ in range(5):
        for (plan, send, recv, _), st in zip(outs, streams):
            plan.launch(send, recv, st)
    torch.cuda.synchronize()
    for plan, send, recv, ref in outs:
        plan.check()
        for a, b in zip(recv, ref):
            assert np.array_equal(a.cpu().numpy(), b)
        plan.close()


@pytest.mark.parametrize("window", ["4096", "65536"])
@pytest.mark.parametrize("name,nbytes", [("ag_777", 1 << 20), ("ar_56_14_14", 1 << 20), ("ag_b7_ring8", 1 << 20),
                                         ("ar_822", 1 << 20), ("ar_ring", 2 << 20), ("rs_ring8", 1 << 20),
                                         ("ar_dgx1", 1 << 20), ("bcast_chain", 1 << 20), ("a2a_k2", 1 << 20)])
def test_window_major_forced(monkeypatch, window, name, nbytes):
    """Window-major execution and the L2 hints (on by default only for
    launches over 1 GB) forced at small sizes, both counter-release modes
    exercised through the tile counts: bit-exact."""
    monkeypatch.setenv("SCCL_WINDOW", window)
    monkeypatch.setenv("SCCL_L2HINT", "1")
    monkeypatch.setenv("SCCL_DISCARD", "1")  # drop consumed scratch receipts from L2
    js = SCHED[name]
    kind = json.loads(js)["collective"]
    dt = O.BF16 if kind in ("allreduce", "reducescatter", "reduce") else O.U8
    run_gpu(js, nbytes, dt, protocol="simple", repeats=2)


def test_auto_plan_switches_per_size():
    """AutoLoopbackPlan over an allgather frontier: each size picks its
    schedule and protocol, results equal the oracle of the chosen schedule."""
    cands = [SCHED["ag_777"], SCHED["ag_b4_oneshot8"], SCHED["ag_b7_ring8"], SCHED["ag_b8_bidir8"]]
    auto = sccl.AutoLoopbackPlan(cands, O.U8, device=0)
    chosen = set()
    for nb in (1024, 65536, 1 << 20, 16 << 20):
        i, proto, plan = auto.plan_for(nb)
        chosen.add((i, proto))
        d = json.loads(cands[i])
        ins = O.seeded_inputs(d["collective"], d["P"], nb, O.U8, nb)
        ref = O.execute(d, ins, nb, O.U8)
        send = [torch.from_numpy(x).to(DEV) for x in ins]
        recv = [torch.zeros(r.size, dtype=torch.uint8, device=DEV) for r in ref]
        torch.cuda.synchronize()
        assert auto.launch(send, recv, nb) == (i, proto)
        torch.cuda.synchronize()
        auto.check()
        for a, b in zip(recv, ref):
            assert np.array_equal(a.cpu().numpy(), b)
    assert len({p for _, p in chosen}) == 2  # LL for the small sizes, the bulk protocol for the large
    auto.close()


def test_baseline_full_sizes():
    """BASELINE configs 2-4 at their largest sizes, through size-independent
    properties: AG (7,7,7) at 1 GiB per rank (every output == the
    concatenation of the inputs), AR (8,2,2) bf16 at 1 GiB with
    integer-valued inputs (exact sum in any order), A2A (8,1,1) at 256 MiB
    (output block s of rank d == input block d of rank s)."""
    P = 8
    g = torch.Generator(device=DEV)
    g.manual_seed(3)
    # allgather, 1 GiB per rank: 8 GiB of inputs, 64 GiB of outputs
    m = 1 << 30
    plan = sccl.LoopbackPlan(SCHED["ag_777"], m, O.U8, device=0)
    send = [torch.randint(0, 256, (m,), dtype=torch.uint8, device=DEV, generator=g) for _ in range(P)]
    recv = [torch.empty(P * m, dtype=torch.uint8, device=DEV) for _ in range(P)]
    plan.launch(send, recv)
    torch.cuda.synchronize()
    plan.check()
    for r in recv:
        for s in range(P):
            assert torch.equal(r[s * m:(s + 1) * m], send[s])
    plan.close()
    del send, recv
    torch.cuda.empty_cache()
    # allreduce (8,2,2), bf16, 1 GiB per rank
    M = 1 << 30
    plan = sccl.LoopbackPlan(SCHED["ar_822"], M, O.BF16, device=0)
    xs = [torch.randint(-16, 17, (M // 2,), device=DEV, generator=g).to(torch.bfloat16) for _ in range(P)]
    recv = [torch.empty(M, dtype=torch.uint8, device=DEV) for _ in range(P)]
    plan.launch([x.view(torch.uint8) for x in xs], recv)
    torch.cuda.synchronize()
    plan.check()
    want = xs[0].float()
    for x in xs[1:]:
        want += x.float()
    want = want.to(torch.bfloat16).view(torch.uint8)
    for r in recv:
        assert torch.equal(r, want)
    plan.close()
    del xs, recv, want
    torch.cuda.empty_cache()
    # alltoall (8,1,1), 256 MiB per rank
    M = 256 << 20
    B = M // P
    plan = sccl.LoopbackPlan(SCHED["a2a_b5"], M, O.U8, device=0)
    send = [torch.randint(0, 256, (M,), dtype=torch.uint8, device=DEV, generator=g) for _ in range(P)]
    recv = [torch.empty(M, dtype=torch.uint8, device=DEV) for _ in range(P)]
    plan.launch(send, recv)
    torch.cuda.synchronize()
    plan.check()
    for d in range(P):
        for s in range(P):
            assert torch.equal(recv[d][s * B:(s + 1) * B], send[s][d * B:(d + 1) * B])
    plan.close()


def test_allreduce_bf16_bitexact_16MiB():
    js = SCHED["ar_56_14_14"]
    run_gpu(js, 16 << 20, O.BF16, seed=9)


def test_unverified_schedule_rejected_on_gpu():
    d = json.loads(SCHED["ag_b4_oneshot8"])
    d["sends"] = d["sends"][1:]
    with pytest.raises(sccl.InvalidArgumentError):
        sccl.LoopbackPlan(d, 4096, O.U8, device=0)


@pytest.mark.parametrize("protocol", ["ll", "simple"])
@pytest.mark.parametrize("name", sorted(SCHED))
def test_both_protocols(name, protocol):
    """LL (flag-in-data) and simple (TMA bulk + counters) on the same cases."""
    js = SCHED[name]
    kind = json.loads(js)["collective"]
    dts = [O.U8] if kind not in ("reduce", "reducescatter", "allreduce") else [O.BF16, O.F32, O.I32]
    for nbytes in (8, 4096 + 48, 40000):
        for dt in dts:
            if nbytes % O.ESIZE[dt] or (kind == "alltoall" and nbytes % (json.loads(js)["P"] * O.ESIZE[dt])):
                continue
            run_gpu(js, nbytes, dt, protocol=protocol, repeats=2)


@pytest.mark.parametrize("kc,kb", [(3, 2), (7, 2)])
def test_chunk_groups_gpu(kc, kb):
    run_gpu(SCHED["ag_777"], 3 * 65536 + 1024, O.U8, nch=kb, kc=kc)
    run_gpu(SCHED["ar_56_14_14"], 3 * 65536 + 1024, O.BF16, nch=kb, kc=kc)
    run_gpu(SCHED["ar_56_14_14"], 24000, O.BF16, nch=kb, kc=kc, protocol="ll", repeats=3)


def test_many_chunk_groups_small():
    """many chunk groups (28 x 8 ranks = 224 CTAs, small tiles; 56 with LL)"""
    run_gpu(SCHED["ag_777"], 20000, O.U8, nch=1, kc=28, protocol="simple", repeats=2)
    run_gpu(SCHED["ar_56_14_14"], 20000, O.F32, nch=1, kc=28, protocol="simple", repeats=2)
    run_gpu(SCHED["ag_777"], 20000, O.U8, nch=1, kc=56, protocol="ll", repeats=2)


SYN = sorted(__import__("glob").glob(__import__("os").path.join(__import__("os").path.dirname(__file__), "golden",
                                                                     "schedules", "*.json")))


@pytest.mark.parametrize("path", SYN, ids=[p.split("/")[-1][:-5] for p in SYN])
@pytest.mark.parametrize("protocol", ["ll", "simple"])
def test_synthesized_schedules_gpu(path, protocol):
    js = open(path).read().strip()
    kind = json.loads(js)["collective"]
    for nb in (8 * 1000, 8 * 65536 + 64):
        for dt in ([O.BF16, O.I32] if kind == "allreduce" else [O.U8]):
            run_gpu(js, nb, dt, protocol=protocol)


def test_topology_discovery_gpu():
    from paper_2008_08708_b200 import topology
    info = topology.discover()
    assert info["devices"] >= 1 and info["target"] != "unknown"
    print("topology:", info)


@pytest.mark.parametrize("name", ["ag_777", "ag_b7_ring8", "a2a_b5", "bcast_chain"])
def test_copy_engine_baseline_matches(name):
    """The copy-engine comparison backend runs the same lowered program."""
    js = SCHED[name]
    d = json.loads(js)
    nb = 1 << 20
    ins = O.seeded_inputs(d["collective"], d["P"], nb, O.U8, 21)
    ref = O.execute(d, ins, nb, O.U8)
    plan = sccl.LoopbackPlan(js, nb, O.U8, device=0, protocol="simple")
    send = [torch.from_numpy(x).to(DEV) for x in ins]
    recv = [torch.zeros(r.size, dtype=torch.uint8, device=DEV) for r in ref]
    plan.launch_copy_engine(send, recv)
    torch.cuda.synchronize()
    for r, (a, b) in enumerate(zip(recv, ref)):
        got = np.where(_covered(d, nb, r, b.size), a.cpu().numpy(), 0)
        assert np.array_equal(got, b)


@pytest.mark.parametrize("dt", [O.F32, O.BF16, O.F16])
@pytest.mark.parametrize("name", ["ar_822", "ar_56_14_14", "ar_ring", "rs_ring8"])
@pytest.mark.parametrize("protocol", ["simple", "ll"])
def test_float_reduction_within_stated_tolerance(name, dt, protocol):
    """Against an order-free reference, the fp64 sum of the same inputs
    (uniform in [-1, 1), not integer-valued): every output element within the
    recursive-summation bound |got - exact| <= P * u * sum_i |x_i|, u = unit
    roundoff of the dtype (f32 2^-24, bf16 2^-8, f16 2^-11) -- P-1 rounded
    adds plus the final rounding, in any order (north_star: "an fp32/bf16
    tolerance stated otherwise").  Bit-exactness against the schedule's own
    order is test_parity_u8_and_float's job."""
    js = SCHED[name]
    d = json.loads(js)
    P = d["P"]
    nbytes = (1 << 20) if protocol == "simple" else (64 << 10)
    npdt = {O.F32: np.float32, O.BF16: None, O.F16: np.float16}[dt]
    u = {O.F32: 2.0 ** -24, O.BF16: 2.0 ** -8, O.F16: 2.0 ** -11}[dt]
    rng = np.random.default_rng(7)
    plan = sccl.LoopbackPlan(js, nbytes, dt, device=0, protocol=protocol)
    n = plan.send_bytes // O.ESIZE[dt]
    xs64 = [rng.uniform(-1, 1, n) for _ in range(P)]
    if dt == O.BF16:  # round to nearest even bf16 via the f32 bit pattern
        ins = []
        for x in xs64:
            b = x.astype(np.float32).view(np.uint32)
            b = ((b + 0x7FFF + ((b >> 16) & 1)) >> 16).astype(np.uint16)
            ins.append(b.view(np.uint8))
        vals = [(x.view(np.uint16).astype(np.uint32) << 16).view(np.float32).astype(np.float64) for x in ins]
    else:
        ins = [x.astype(npdt).view(np.uint8) for x in xs64]
        vals = [x.view(npdt).astype(np.float64) for x in ins]
    exact = np.sum(vals, axis=0)
    bound = P * u * np.sum(np.abs(vals), axis=0)
    send = [torch.from_numpy(np.ascontiguousarray(x)).to(DEV) for x in ins]
    recv = [torch.zeros(plan.recv_bytes, dtype=torch.uint8, device=DEV) for _ in range(P)]
    plan.launch(send, recv)
    torch.cuda.synchronize()
    plan.check()
    geo_sz = plan.recv_bytes // O.ESIZE[dt]
    plan.close()
    for r in range(P):
        raw = recv[r].cpu().numpy()
        if dt == O.BF16:
            got = (raw.view(np.uint16).astype(np.uint32) << 16).view(np.float32).astype(np.float64)
        else:
            got = raw.view(npdt).astype(np.float64)
        if d["collective"] == "reducescatter":  # rank r holds block r of the sum
            want, bnd = exact[r * geo_sz:(r + 1) * geo_sz], bound[r * geo_sz:(r + 1) * geo_sz]
        else:
            want, bnd = exact, bound
        err = np.abs(got - want)
        assert np.all(err <= bnd), (r, float(np.max(err - bnd)))


@pytest.mark.parametrize("protocol", ["ll", "simple"])
@pytest.mark.parametrize("dt", [O.I32, O.F32, O.BF16])
def test_dgx1_48_6_14_direct_sum(protocol, dt):
    """SPEC.md:426 / acceptance :641 on the GPU: the DGX-1 Allreduce
    (48,6,14) (RS+AG of the synthesized (6,3,7)) over random integer
    payloads leaves all 8 ranks with the direct sum, bit for bit (for the
    float types: integer values in [-16, 16], exact in any order), and
    equal to the oracle."""
    js = open(__import__("os").path.join(__import__("os").path.dirname(__file__), "golden", "schedules",
                                         "ar_from_dgx1_6_3_7.json")).read().strip()
    d = json.loads(js)
    assert (d["C"], d["S"], d["R"]) == (48, 6, 14)
    nbytes = 48 * 4096 if protocol == "simple" else 48 * 256
    mode = "random" if dt == O.I32 else "smallint"
    ins = O.seeded_inputs("allreduce", 8, nbytes, dt, 641, mode)
    npdt = {O.I32: np.int32, O.F32: np.float32}.get(dt)
    if dt == O.BF16:
        vals = [(x.view(np.uint16).astype(np.uint32) << 16).view(np.float32).astype(np.float64) for x in ins]
    else:
        vals = [x.view(npdt).astype(np.float64 if dt != O.I32 else np.int64) for x in ins]
    direct = np.sum(vals, axis=0)
    ref = O.execute(d, ins, nbytes, dt)
    run_gpu(js, nbytes, dt, seed=641, mode=mode, protocol=protocol)
    for o in ref:
        if dt == O.BF16:
            got = (o.view(np.uint16).astype(np.uint32) << 16).view(np.float32).astype(np.float64)
        elif dt == O.I32:
            got = o.view(np.int32).astype(np.int64)
            direct = direct.astype(np.int64).astype(np.int32).astype(np.int64)  # wrapping sum
        else:
            got = o.view(npdt).astype(np.float64)
        assert np.array_equal(got, direct)


def test_auto_plan_from_machine_gpu():
    """Topology discovery on this box (one GPU: loopback) -> the committed
    frontiers for P = 8 -> the cost model's per-size choice: allgather and
    allreduce at several sizes, bit-exact with the oracle."""
    for coll, dt in (("allgather", O.U8), ("allreduce", O.BF16)):
        ap = sccl.AutoLoopbackPlan.from_machine(coll, 8, dt)
        assert ap.discovery["target"] == "loopback:1"
        chosen = set()
        for nb in (1024, 64 << 10, 4 << 20):
            i, proto, plan = ap.plan_for(nb)
            chosen.add((i, proto))
            d = json.loads(ap.schedules[i])
            ins = O.seeded_inputs(coll, 8, nb, dt, 3)
            ref = O.execute(d, ins, nb, dt)
            send = [torch.from_numpy(x).to(DEV) for x in ins]
            recv = [torch.zeros(r.size, dtype=torch.uint8, device=DEV) for r in ref]
            ap.launch(send, recv, nb)
            torch.cuda.synchronize()
            ap.check()
            assert all(np.array_equal(a.cpu().numpy(), b) for a, b in zip(recv, ref)), (coll, nb)
        assert len(chosen) >= 2, chosen  # the choice changes with size
        ap.close()


FRONTIER_DIR = os.path.join(os.path.dirname(S.__file__), "frontiers")
FRONTIERS = sorted(f[:-5] for f in os.listdir(FRONTIER_DIR) if f.endswith(".json") and f != "index.json")


@pytest.mark.parametrize("name", FRONTIERS)
@pytest.mark.parametrize("protocol", ["ll", "simple"])
def test_every_committed_frontier_schedule(name, protocol):
    """Every Pareto-frontier schedule shipped in frontiers/ (ring(P), full(P)
    and the NVSwitch target switch(P), P = 2/4/8; SURVEY.md 8(d) cfg 5):
    the allgather itself and the allreduce composed from it (RS = its
    inversion, bf16), bit-exact against the oracle under both protocols,
    sentinel-checked."""
    with open(os.path.join(FRONTIER_DIR, name + ".json")) as f:
        js = f.read()
    run_gpu(js, 24576 + 48, O.U8, seed=61, protocol=protocol)
    run_gpu(S.allreduce_from(json.loads(js)), 8 * 4096, O.BF16, seed=62, protocol=protocol)


BENCH_FILES = sorted(__import__("glob").glob(os.path.join(os.path.dirname(__file__), "golden", "schedules", "bench",
                                                          "*.json")))


@pytest.mark.parametrize("path", BENCH_FILES, ids=[p.split("/")[-1][:-5] for p in BENCH_FILES])
def test_bench_schedule_files_gpu(path):
    """Every schedule file bench.py runs (N = 1 loopback and the N = 2/4/8
    workloads, NCCL comparisons and sweeps, P = 1 self-test files included),
    executed in loopback at a small size, bit-exact against the oracle."""
    js = open(path).read().strip()
    d = json.loads(js)
    dt = O.BF16 if d["collective"] == "allreduce" else O.U8
    nb = 4096 * max(1, d["P"])
    for protocol in ("ll", "simple"):
        run_gpu(js, nb, dt, seed=71, protocol=protocol)
