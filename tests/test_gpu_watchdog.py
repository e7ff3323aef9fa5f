"""The watchdog's cooperative abort (status 5, peer
timeout; /root/reference/proj/include/sccl/error.hpp:9-30).

Two processes, one rank each, on cuda:0; rank 1 binds but never launches.
Rank 0's launch must end on its own after timeout_ms (no trap, no hang),
sccl_plan_check must return SCCL_PEER_TIMEOUT, the poisoned plan must refuse
the next launch with the same status, and the CUDA context must still run
work afterwards: a torch kernel and a fresh loopback plan checked against
the oracle."""
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKER = r"""
import json, sys, time
sys.path[:0] = [{root!r}, {oracle!r}]
import numpy as np, torch, torch.distributed as dist
import oracle as O
from paper_2008_08708_b200 import sccl, schedules as S
rank, proto = int(sys.argv[1]), sys.argv[2]
dist.init_process_group("gloo", init_method="tcp://127.0.0.1:{port}", rank=rank, world_size=2)
torch.cuda.set_device(0)
js = S.allreduce_from(S.one_shot_allgather(2))
nb = 1 << 20 if proto == "simple" else 8192
plan = sccl.Plan(js, rank, 2, nb, O.BF16, device=0, protocol=proto, timeout_ms=500)
plan.bind_with()
if rank == 0:
    send = torch.zeros(nb, dtype=torch.uint8, device="cuda")
    recv = torch.zeros(nb, dtype=torch.uint8, device="cuda")
    t0 = time.time()
    plan.launch(send, recv)
    torch.cuda.synchronize()  # must return: the kernel aborts, it does not trap or hang
    dt = time.time() - t0
    try:
        plan.check()
        raise SystemExit("watchdog did not fire")
    except sccl.PeerTimeoutError as e:
        assert e.code == sccl.PEER_TIMEOUT and "peer timeout" in str(e), str(e)
    try:
        plan.launch(send, recv)
        raise SystemExit("poisoned plan launched")
    except sccl.PeerTimeoutError as e:
        assert e.code == sccl.PEER_TIMEOUT
    # the context is alive: a torch kernel and a fresh loopback plan
    assert float(torch.ones(1 << 20, device="cuda").sum()) == float(1 << 20)
    d = json.loads(S.allreduce_from(S.one_shot_allgather(8)))
    ins = O.seeded_inputs("allreduce", 8, 65536, O.F32, 5)
    ref = O.execute(d, ins, 65536, O.F32)
    lp = sccl.LoopbackPlan(json.dumps(d), 65536, O.F32, device=0, protocol=proto)
    s2 = [torch.from_numpy(x).cuda() for x in ins]
    r2 = [torch.zeros(65536, dtype=torch.uint8, device="cuda") for _ in range(8)]
    lp.launch(s2, r2)
    torch.cuda.synchronize()
    lp.check()
    assert all(np.array_equal(a.cpu().numpy(), b) for a, b in zip(r2, ref))
    lp.close()
    print(f"ABORTED_OK {{proto}} {{dt:.2f}}s", flush=True)
dist.barrier()
plan.close()
dist.destroy_process_group()
"""


@pytest.mark.parametrize("proto", ["simple", "ll"])
def test_peer_timeout_aborts_cooperatively(tmp_path, proto):
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    script = tmp_path / "w.py"
    script.write_text(WORKER.format(root=ROOT, oracle=os.path.join(ROOT, "oracle"), port=port))
    procs = [subprocess.Popen([sys.executable, str(script), str(r), proto], stdout=subprocess.PIPE,
                              stderr=subprocess.PIPE, text=True) for r in range(2)]
    try:
        outs = [p.communicate(timeout=240) for p in procs]
    finally:
        for p in procs:
            if p.poll() is None:
                p.kill()
    for p, (o, e) in zip(procs, outs):
        assert p.returncode == 0, (o, e[-3000:])
    assert "ABORTED_OK" in outs[0][0], outs
    secs = float(outs[0][0].split()[-1].rstrip("s"))
    assert secs < 30, f"abort took {secs} s"
