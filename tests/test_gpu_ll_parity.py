"""Epoch-parity LL slot sets (plan.cpp ll_parity_safe): one-rank-per-process
LL plans whose schedule makes every receiver part of every sender's
completion set skip the entry handshake and alternate two scratch slot sets
by launch parity.  The hazard this replaces the handshake for -- a sender
overwriting a slot its receiver has not read yet -- only shows when ranks
drift apart, so here the ranks launch many times back to back with NO
barrier or synchronize between launches, one rank stalling its host thread
at random, every launch with its own input and output; every output is then
compared with the CPU oracle.  The same harness runs the kinds that keep the
handshake (broadcast) and, with SCCL_LL_PARITY=0, the handshake variant of
the parity-eligible kinds.  Processes share cuda:0 (time-sliced contexts)."""
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKER = r"""
import json, os, random, sys, time
sys.path[:0] = [{root!r}, {oracle!r}]
import numpy as np, torch, torch.distributed as dist
import oracle as O
from paper_2008_08708_b200 import sccl, schedules as S
rank, W, MEM, N = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], int(sys.argv[4])
dist.init_process_group("gloo", init_method="tcp://127.0.0.1:{port}", rank=rank, world_size=W)
torch.cuda.set_device(0)
cases = [
    ("ag_oneshot", S.to_json(S.one_shot_allgather(W)), 4096 + 48, O.U8, 1),
    ("ag_ring", S.to_json(S.ring_allgather(W)), 8192, O.U8, 1),
    ("a2a", S.to_json(S.direct_alltoall(W)), 1024 * W, O.U8, 1),
    ("ar_oneshot", S.allreduce_from(S.one_shot_allgather(W)), 4096, O.BF16, 1),
    ("ar_ring", S.allreduce_from(S.ring_allgather(W)), 8192, O.F32, 1),
    ("bcast", S.to_json(S.one_shot_broadcast(W)), 4096, O.U8, 0),  # rooted: keeps the handshake
]
rng = random.Random(1234 + rank)
for name, js, nb, dt, want_parity in cases:
    d = json.loads(js)
    plan = sccl.Plan(js, rank, W, nb, dt, device=0, protocol="ll", timeout_ms=120000, mem_handles=MEM)
    info = plan.info()
    parity_env = os.environ.get("SCCL_LL_PARITY") != "0"
    assert info["ll_parity"] == (1 if (want_parity and parity_env) else 0), (name, info["ll_parity"])
    plan.bind_with()
    ins = [O.seeded_inputs(d["collective"], W, nb, dt, 100 + i) for i in range(N)]
    refs = [O.execute(d, x, nb, dt)[rank] for x in ins]
    sends = [torch.from_numpy(x[rank]).cuda() for x in ins]
    recvs = [torch.full((r.size,), 0xEE, dtype=torch.uint8, device="cuda") for r in refs]
    torch.cuda.synchronize()
    dist.barrier()
    for i in range(N):  # back to back: no barrier, no synchronize
        if rank == 0 and rng.random() < 0.3:
            time.sleep(rng.random() * 0.002)  # this rank's launches drift behind its peers'
        plan.launch(sends[i], recvs[i])
    torch.cuda.synchronize()
    plan.check()
    bad = [i for i in range(N) if not np.array_equal(recvs[i].cpu().numpy(), refs[i])]
    assert not bad, (name, "launches differ from the oracle", bad[:10])
    dist.barrier()
    plan.close()
    print("OK", rank, name, info["ll_parity"], flush=True)
# registered (zero-copy) receive buffers: receipts still land in the parity
# slot sets and the receiver unpacks into each launch's own registered target
js = S.allreduce_from(S.ring_allgather(W))
d = json.loads(js)
nb, K = 8192, 8
plan = sccl.Plan(js, rank, W, nb, O.F32, device=0, protocol="ll", timeout_ms=120000, mem_handles=MEM)
plan.bind_with()
targets = [torch.full((nb,), 0xEE, dtype=torch.uint8, device="cuda") for _ in range(K)]
for t in targets:
    plan.register(t)
ins = [O.seeded_inputs("allreduce", W, nb, O.F32, 300 + i) for i in range(K)]
refs = [O.execute(d, x, nb, O.F32)[rank] for x in ins]
sends = [torch.from_numpy(x[rank]).cuda() for x in ins]
torch.cuda.synchronize()
dist.barrier()
for i in range(K):
    if rank == 0 and rng.random() < 0.5:
        time.sleep(rng.random() * 0.002)
    plan.launch(sends[i], targets[i])
torch.cuda.synchronize()
plan.check()
bad = [i for i in range(K) if not np.array_equal(targets[i].cpu().numpy(), refs[i])]
assert not bad, ("registered", bad)
dist.barrier()
plan.close()
print("OK", rank, "registered", flush=True)
# CUDA-graph replays: the slot-set parity comes from the device-side launch
# epoch, so a captured launch replayed many times keeps alternating sets;
# 5 captured launches (odd, so consecutive replays start on different sets),
# replayed 3 times back to back, ranks drifting; the last output is checked
js = S.to_json(S.ring_allgather(W))
d = json.loads(js)
nb = 4096
plan = sccl.Plan(js, rank, W, nb, O.U8, device=0, protocol="ll", timeout_ms=120000, mem_handles=MEM)
plan.bind_with()
x = O.seeded_inputs("allgather", W, nb, O.U8, 900)
want = O.execute(d, x, nb, O.U8)[rank]
send = torch.from_numpy(x[rank]).cuda()
recv = torch.full((want.size,), 0xEE, dtype=torch.uint8, device="cuda")
st = torch.cuda.Stream()
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=st):
    for _ in range(5):
        plan.launch(send, recv, st)
dist.barrier()
with torch.cuda.stream(st):
    for _ in range(3):
        if rank == 0:
            time.sleep(rng.random() * 0.002)
        g.replay()
torch.cuda.synchronize()
plan.check()
assert np.array_equal(recv.cpu().numpy(), want), ("graph", rank)
dist.barrier()
plan.close()
print("OK", rank, "graph", flush=True)
dist.destroy_process_group()
"""


CASES = [(w, m, par) for w in (2, 4) for m in ("ipc", "vmm") for par in ("on", "off")] + [(8, "ipc", "on")]


@pytest.mark.parametrize("world,mem,parity", CASES, ids=[f"w{w}-{m}-{par}" for w, m, par in CASES])
def test_ll_back_to_back_without_barriers(tmp_path, world, mem, parity):
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    script = tmp_path / "w.py"
    script.write_text(WORKER.format(root=ROOT, oracle=os.path.join(ROOT, "oracle"), port=port))
    env = dict(os.environ, MASTER_ADDR="127.0.0.1")
    if parity == "off":
        env["SCCL_LL_PARITY"] = "0"
    else:
        env.pop("SCCL_LL_PARITY", None)
    n = "40"
    procs = [subprocess.Popen([sys.executable, str(script), str(r), str(world), mem, n], stdout=subprocess.PIPE,
                              stderr=subprocess.PIPE, text=True, env=env) for r in range(world)]
    try:
        outs = [p.communicate(timeout=600) for p in procs]
    finally:
        for p in procs:
            if p.poll() is None:
                p.kill()
    for p, (o, e) in zip(procs, outs):
        assert p.returncode == 0, (o, e[-3000:])
    assert "".join(o for o, _ in outs).count("OK") == 8 * world
