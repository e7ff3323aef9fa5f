"""One rank per GPU over NVLink / NVSwitch: the configuration north_star is
about.  Runs when at least two CUDA
devices are visible: W = device count (up to 8) processes, rank r on cuda:r,
peers' plan regions mapped through CUDA IPC handles and through VMM (cuMem
POSIX fds).  Every rank's output must equal the CPU oracle bit for bit
(4 KiB and 1 MiB per rank), or, at 64 MiB, satisfy the size-independent
properties (allgather = concatenation of the inputs; allreduce of
integer-valued floats = the exact sum in any order), under both protocols,
with back-to-back launches (entry handshake, epochs).

Covered pieces that a single device cannot exercise: cp.async.bulk stores
into a peer-mapped region, fence.release.sys ordering of those async-proxy
writes over NVLink, cross-device cuMemSetAccess, LL words over NVLink.

With fewer than two devices the test skips.  SCCL_MULTIDEVICE_SHARE=1 runs
the same harness with every rank on cuda:0 (validates the harness itself on
a one-GPU box; the contexts time-slice)."""
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHARE = os.environ.get("SCCL_MULTIDEVICE_SHARE") == "1"

WORKER = r"""
import json, os, sys
sys.path[:0] = [{root!r}, {oracle!r}]
import numpy as np, torch, torch.distributed as dist
import oracle as O
from paper_2008_08708_b200 import sccl, schedules as S
rank, W, MEM, SHARE = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], sys.argv[4] == "1"
dist.init_process_group("gloo", init_method="tcp://127.0.0.1:{port}", rank=rank, world_size=W)
dev = 0 if SHARE else rank
torch.cuda.set_device(dev)
# SCCL_MULTIDEVICE_NCH: CTAs per rank (0 = policy).  Under MPS the shared-GPU
# ranks run concurrently and must be co-resident together (W x CTAs <= SM slots)
NCH = int(os.environ.get("SCCL_MULTIDEVICE_NCH", "0"))
ag1 = S.one_shot_allgather(W)
scheds = [("ag111", S.to_json(ag1), [O.U8]),
          ("ag_ring", S.to_json(S.ring_allgather(W)), [O.U8]),
          ("ar_oneshot", S.allreduce_from(ag1), [O.BF16, O.F32]),
          ("a2a", S.to_json(S.direct_alltoall(W)), [O.U8])]
if W not in (4, 6):  # K_4* and K_6* have no Hamiltonian decomposition
    ham = S.hamiltonian_allgather(W)
    scheds += [("ag_ham", S.to_json(ham), [O.U8]), ("ar_ham", S.allreduce_from(ham), [O.BF16, O.F32])]
sizes = [4096, 1 << 20] + ([] if SHARE else [64 << 20])
n_ok = 0
for name, js, dts in scheds:
    d = json.loads(js)
    kind = d["collective"]
    for dt in dts:
        for nb in sizes:
            for proto in ("ll", "simple"):
                if proto == "ll" and nb > (1 << 20):
                    continue
                plan = sccl.Plan(js, rank, W, nb, dt, device=dev, protocol=proto, timeout_ms=120000, nchannels=NCH,
                                 mem_handles=MEM)
                plan.bind_with()
                for it in range(3):  # back-to-back: entry handshake + epochs advance
                    if nb <= (1 << 20):
                        ins = O.seeded_inputs(kind, W, nb, dt, 23 + it)
                        want = O.execute(d, ins, nb, dt)[rank]
                        send = torch.from_numpy(ins[rank]).cuda()
                    else:  # property checks at full size
                        g = torch.Generator(device="cuda")
                        xs = []
                        for r in range(W):
                            g.manual_seed(1000 * it + r)
                            if kind == "allreduce":
                                tdt = torch.bfloat16 if dt == O.BF16 else torch.float32
                                xs.append(torch.randint(-16, 17, (nb // O.ESIZE[dt],), device="cuda",
                                                        generator=g).to(tdt))
                            else:
                                xs.append(torch.randint(0, 256, (nb,), dtype=torch.uint8, device="cuda",
                                                        generator=g))
                        send = xs[rank].view(torch.uint8)
                        if kind == "allgather":
                            want = torch.cat(xs)
                        elif kind == "allreduce":
                            want = torch.stack([x.double() for x in xs]).sum(0).to(xs[0].dtype).view(torch.uint8)
                        else:  # alltoall: block r of my output = block rank of rank r's input
                            blk = nb // W
                            want = torch.cat([xs[r][rank * blk:(rank + 1) * blk] for r in range(W)])
                    recv = torch.full((plan.recv_bytes,), 0xEE, dtype=torch.uint8, device="cuda")
                    plan.launch(send, recv)
                    torch.cuda.synchronize()
                    plan.check()
                    got = recv.cpu().numpy() if nb <= (1 << 20) else recv
                    ok = np.array_equal(got, want) if nb <= (1 << 20) else bool(torch.equal(got, want))
                    assert ok, (name, dt, nb, proto, it, rank)
                    dist.barrier()
                plan.close()
                n_ok += 1
# bursts: 12 launches back to back, no barrier or synchronize between them,
# each with its own input and output (LL: the epoch-parity slot sets; simple:
# the entry handshake into the peers' receive buffers), then every output
# against the oracle
for name, js, dts in scheds:
    d = json.loads(js)
    for proto, nb in (("ll", 4096), ("simple", 1 << 18)):
        plan = sccl.Plan(js, rank, W, nb, dts[0], device=dev, protocol=proto, timeout_ms=120000, mem_handles=MEM,
                         nchannels=NCH)
        plan.bind_with()
        ins = [O.seeded_inputs(d["collective"], W, nb, dts[0], 500 + i) for i in range(12)]
        wants = [O.execute(d, x, nb, dts[0])[rank] for x in ins]
        sends = [torch.from_numpy(x[rank]).cuda() for x in ins]
        recvs = [torch.full((plan.recv_bytes,), 0xEE, dtype=torch.uint8, device="cuda") for _ in ins]
        torch.cuda.synchronize()
        dist.barrier()
        for sb, rb in zip(sends, recvs):
            plan.launch(sb, rb)
        torch.cuda.synchronize()
        plan.check()
        bad = [i for i, (rb, w) in enumerate(zip(recvs, wants)) if not np.array_equal(rb.cpu().numpy(), w)]
        assert not bad, ("burst", name, proto, rank, bad)
        dist.barrier()
        plan.close()
        n_ok += 1
# torch symmetric memory as the plan region (one rank per GPU)
if MEM == "ipc" and not SHARE:
    for name, js, dts in scheds[:3]:
        d = json.loads(js)
        for proto in ("ll", "simple"):
            nb = 1 << 20
            plan = sccl.Plan(js, rank, W, nb, dts[0], device=dev, protocol=proto, timeout_ms=120000,
                             mem_handles="external")
            plan.bind_symmetric_memory()
            ins = O.seeded_inputs(d["collective"], W, nb, dts[0], 77)
            want = O.execute(d, ins, nb, dts[0])[rank]
            recv = torch.full((plan.recv_bytes,), 0xEE, dtype=torch.uint8, device="cuda")
            plan.launch(torch.from_numpy(ins[rank]).cuda(), recv)
            torch.cuda.synchronize()
            plan.check()
            assert np.array_equal(recv.cpu().numpy(), want), ("symm_mem", name, proto, rank)
            dist.barrier()
            plan.close()
            n_ok += 1
print("OK", rank, n_ok, flush=True)
dist.destroy_process_group()
"""


def _world():
    n = torch.cuda.device_count() if torch.cuda.is_available() else 0
    if SHARE and n >= 1:
        return int(os.environ.get("SCCL_MULTIDEVICE_WORLD", "2"))
    return min(n, 8)


def _run(tmp_path, W, mem, share):
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    script = tmp_path / "w.py"
    script.write_text(WORKER.format(root=ROOT, oracle=os.path.join(ROOT, "oracle"), port=port))
    procs = [subprocess.Popen([sys.executable, str(script), str(r), str(W), mem, "1" if share else "0"],
                              stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True) for r in range(W)]
    try:
        outs = [p.communicate(timeout=1700) for p in procs]
    finally:
        for p in procs:
            if p.poll() is None:
                p.kill()
    for p, (o, e) in zip(procs, outs):
        assert p.returncode == 0, (o, e[-3000:])
    assert sum("OK" in o for o, _ in outs) == W


@pytest.mark.timeout(1800)
@pytest.mark.parametrize("mem", ["ipc", "vmm"])
def test_one_rank_per_gpu(tmp_path, mem):
    W = _world()
    if W < 2:
        pytest.skip(f"one rank per GPU needs >= 2 CUDA devices, {W} visible (set SCCL_MULTIDEVICE_SHARE=1 "
                    "to run the harness with every rank on cuda:0)")
    _run(tmp_path, W, mem, SHARE)


@pytest.mark.timeout(1800)
def test_eight_rank_processes_time_sliced_on_one_gpu(tmp_path):
    """The 8-rank multi-process configuration of the 8 x B200 box (every P=8
    schedule the bench uses, (7,7,7) and (56,14,14) included) with eight
    processes -- eight CUDA contexts, IPC-mapped regions, sys-scope
    counters, entry handshakes -- all on cuda:0.  Correctness only (the
    contexts time-slice); runs on any box with a GPU."""
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    _run(tmp_path, 8, "ipc", True)
