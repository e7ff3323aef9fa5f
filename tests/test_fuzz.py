"""Randomized valid schedules (multi-hop trees, uneven fan-in/fan-out) and
their inverted / composed combining forms: lowering interpreter vs the
oracle on CPU, the kernels vs the oracle on GPU."""
import json
import random

import numpy as np
import pytest

import oracle as O
from paper_2008_08708_b200 import sccl
from paper_2008_08708_b200 import schedules as S


def _cases(n, seed0):
    rng = random.Random(seed0)
    out = []
    for i in range(n):
        P = rng.choice([2, 3, 4, 5, 8])
        C = rng.choice([1, 2, 3])
        St = rng.randint(1, 4)
        ag = json.dumps(S.random_allgather(P, C, St, seed=seed0 * 1000 + i))
        ag = sccl.canonicalize(ag)
        kind = rng.choice(["ag", "rs", "ar"])
        js = ag if kind == "ag" else sccl.invert(ag) if kind == "rs" else sccl.compose_allreduce(sccl.invert(ag), ag)
        dt = O.U8 if kind == "ag" else rng.choice([O.I32, O.F32, O.BF16, O.F16])
        nb = rng.choice([16, 100 * O.ESIZE[dt], 4096, 12000 + 16 * rng.randint(0, 100)])
        nb -= nb % O.ESIZE[dt]
        out.append((js, nb, dt, rng.choice(["ll", "simple"]), rng.choice([(0, 0), (2, 3), (1, 1)])))
    return out


@pytest.mark.parametrize("case", range(60))
def test_fuzz_interpreter(case):
    js, nb, dt, proto, (kc, kb) = _cases(60, 1)[case]
    d = json.loads(js)
    assert sccl.verify(js) == [] and O.verify(d) == []
    ins = O.seeded_inputs(d["collective"], d["P"], nb, dt, case)
    ref = O.execute(d, ins, nb, dt)
    ref2 = O.execute_py(d, ins, nb, dt)
    assert all(np.array_equal(a, b) for a, b in zip(ref, ref2))
    p = sccl.LoopbackPlan(js, nb, dt, device=-1, protocol=proto, chunk_groups=kc, nchannels=kb,
                          tile_bytes=256 if proto == "simple" else 0)
    outs = [np.zeros_like(r) for r in ref]
    p.interpret_on_cpu(ins, outs)
    for a, b in zip(outs, ref):
        assert np.array_equal(a, b)


@pytest.mark.gpu
@pytest.mark.parametrize("case", range(40))
def test_fuzz_gpu(case):
    import torch
    js, nb, dt, proto, (kc, kb) = _cases(40, 2)[case]
    d = json.loads(js)
    ins = O.seeded_inputs(d["collective"], d["P"], nb, dt, case)
    ref = O.execute(d, ins, nb, dt)
    p = sccl.LoopbackPlan(js, nb, dt, device=0, protocol=proto, chunk_groups=kc, nchannels=kb)
    send = [torch.from_numpy(x).cuda() for x in ins]
    recv = [torch.zeros(r.size, dtype=torch.uint8, device="cuda") for r in ref]
    for _ in range(2):
        p.launch(send, recv)
    torch.cuda.synchronize()
    p.check()
    for a, b in zip(recv, ref):
        assert np.array_equal(a.cpu().numpy(), b)
