"""Multi-process path on ONE GPU: two (or four) processes, one rank each,
all on cuda:0.  Exercises exactly what an 8xB200 run uses -- CUDA-IPC export /
bind of the plan regions through torch.distributed (gloo), sys-scope
counters, the per-(peer, channel) entry handshake, the registered receive
buffer and its copy-out -- except that the peer is the same device (the
contexts time-slice instead of running concurrently, so this checks
correctness, not speed)."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKER = r"""
import json, os, sys
sys.path[:0] = [{root!r}, {oracle!r}]
import numpy as np, torch, torch.distributed as dist
import oracle as O
from paper_2008_08708_b200 import sccl, schedules as S
rank, W = int(sys.argv[1]), int(sys.argv[2])
MEM = sys.argv[3] if len(sys.argv) > 3 else "ipc"
dist.init_process_group("gloo", init_method="tcp://127.0.0.1:{port}", rank=rank, world_size=W)
torch.cuda.set_device(0)
if W == 2:
    cases = [
        (S.to_json(S.one_shot_allgather(2)), 1 << 16, O.U8, "simple"),
        (S.to_json(S.one_shot_allgather(2)), 4096, O.U8, "ll"),
        (S.allreduce_from(S.one_shot_allgather(2)), 1 << 18, O.BF16, "simple"),
        (S.allreduce_from(S.one_shot_allgather(2)), 2048, O.F32, "ll"),
        # > 16 tiles per CTA: counters released by the windowed signaler warp
        (S.to_json(S.one_shot_allgather(2)), 32 << 20, O.U8, "simple"),
    ]
else:  # multi-hop relays and combining trees through IPC-mapped peers
    cases = [
        (S.to_json(S.ring_allgather(4)), 1 << 16, O.U8, "simple"),
        (S.allreduce_from(S.recursive_doubling_ring4()), 1 << 16, O.F32, "simple"),
        (S.to_json(S.direct_alltoall(4)), 4096, O.U8, "ll"),
        (S.allreduce_from(S.ring_allgather(4)), 8192, O.BF16, "ll"),
        (S.to_json(S.ring_allgather(4)), 8 << 20, O.U8, "simple"),  # windowed signaler, sys scope
        # chunk % kc would put each rank's alltoall chunks in one group: the
        # balanced chunk-group map, computed independently in every process
        (S.to_json(S.direct_alltoall(4)), 1 << 20, O.U8, "simple"),
        # window-major + L2 hints + receipt discards forced (sys scope)
        ("FORCE", S.allreduce_from(S.one_shot_allgather(4)), 4 << 20, O.BF16, "simple"),
    ]
for case in cases:
    forced = case[0] == "FORCE"
    js, nb, dt, proto = case[1:] if forced else case
    for k, v in (("SCCL_WINDOW", "65536"), ("SCCL_L2HINT", "1"), ("SCCL_DISCARD", "1")):
        if forced:
            os.environ[k] = v
        else:
            os.environ.pop(k, None)
    d = json.loads(js)
    ins = O.seeded_inputs(d["collective"], W, nb, dt, 17)
    ref = O.execute(d, ins, nb, dt)
    plan = sccl.Plan(js, rank, W, nb, dt, device=0, protocol=proto, timeout_ms=120000, mem_handles=MEM)
    plan.bind_with()
    send = torch.from_numpy(ins[rank]).cuda()
    for it in range(3):  # back-to-back launches: entry handshake + epochs
        recv = torch.zeros(ref[rank].size, dtype=torch.uint8, device="cuda")
        plan.launch(send, recv)
        torch.cuda.synchronize()
        plan.check()
        assert np.array_equal(recv.cpu().numpy(), ref[rank]), (d["collective"], proto, it)
        dist.barrier()
    plan.close()
    print("OK", rank, d["collective"], proto, flush=True)
# caller buffers registered as zero-copy receive targets (peers write them
# directly, no copy-out): a slice at an offset inside a larger torch
# allocation, and an in-place allreduce (sendbuf == recvbuf == registered)
for proto in ("simple", "ll"):
    js = S.allreduce_from(S.one_shot_allgather(W)) if W == 2 else S.allreduce_from(S.ring_allgather(W))
    nb = (1 << 20) if proto == "simple" else 8192
    d = json.loads(js)
    plan = sccl.Plan(js, rank, W, nb, O.F32, device=0, protocol=proto, timeout_ms=120000, mem_handles=MEM)
    plan.bind_with()
    big = torch.zeros(nb + 8192, dtype=torch.uint8, device="cuda")
    target = big[4096:4096 + nb]
    plan.register(target)
    inplace = torch.zeros(nb, dtype=torch.uint8, device="cuda")
    plan.register(inplace)
    for it in range(3):
        ins = O.seeded_inputs("allreduce", W, nb, O.F32, 30 + it)
        ref = O.execute(d, ins, nb, O.F32)
        send = torch.from_numpy(ins[rank]).cuda()
        target.fill_(0xEE)
        plan.launch(send, target)
        torch.cuda.synchronize()
        plan.check()
        assert np.array_equal(target.cpu().numpy(), ref[rank]), ("registered", proto, it)
        assert int(big[:4096].max()) == 0 and int(big[4096 + nb:].max()) == 0, "wrote outside the registered slice"
        inplace.copy_(send)
        torch.cuda.synchronize()
        dist.barrier()
        plan.launch(inplace, inplace)
        torch.cuda.synchronize()
        plan.check()
        assert np.array_equal(inplace.cpu().numpy(), ref[rank]), ("in-place registered", proto, it)
        dist.barrier()
    plan.deregister(target)
    plan.close()
    print("OK", rank, "registered", proto, flush=True)
# caller-provided plan regions (mem_handles="external"): torch symmetric
# memory refuses two ranks on one device ("detected allocations from
# overlapping devices"), so here the regions are raw cudaMalloc allocations
# shared with cudaIpcGetMemHandle / cudaIpcOpenMemHandle (the CUDA runtime
# called directly through ctypes); test_gpu_multidevice.py binds torch
# symmetric memory with one rank per GPU
import ctypes, glob
import nvidia.cuda_runtime as _crt
rt = ctypes.CDLL(glob.glob(os.path.join(_crt.__path__[0], "lib", "libcudart.so*"))[0])
class IpcHandle(ctypes.Structure):  # cudaIpcMemHandle_t, passed by value
    _fields_ = [("reserved", ctypes.c_char * 64)]
rt.cudaIpcGetMemHandle.argtypes = [ctypes.POINTER(IpcHandle), ctypes.c_void_p]
rt.cudaIpcOpenMemHandle.argtypes = [ctypes.POINTER(ctypes.c_void_p), IpcHandle, ctypes.c_uint]
js = S.allreduce_from(S.one_shot_allgather(W)) if W == 2 else S.to_json(S.ring_allgather(W))
d = json.loads(js)
nb = 1 << 18
dt = O.BF16 if d["collective"] == "allreduce" else O.U8
for proto in ("simple", "ll"):
    plan = sccl.Plan(js, rank, W, nb, dt, device=0, protocol=proto, timeout_ms=120000, mem_handles="external")
    how, opened, mine = "cuda_ipc", [], ctypes.c_void_p(0)
    if True:  # (symmetric memory: test_gpu_multidevice.py, one rank per GPU)
        assert rt.cudaMalloc(ctypes.byref(mine), ctypes.c_size_t(plan.region_bytes())) == 0
        h = IpcHandle()
        rc = rt.cudaIpcGetMemHandle(ctypes.byref(h), mine)
        assert rc == 0, ("cudaIpcGetMemHandle", rc)
        handles = [None] * W
        dist.all_gather_object(handles, ctypes.string_at(ctypes.addressof(h), 64))  # (.reserved stops at a NUL)
        ptrs = []
        for r in range(W):
            if r == rank:
                ptrs.append(mine.value)
                continue
            q = ctypes.c_void_p(0)
            hr = IpcHandle()
            ctypes.memmove(ctypes.byref(hr), handles[r], 64)
            rc = rt.cudaIpcOpenMemHandle(ctypes.byref(q), hr, 1)
            assert rc == 0, ("cudaIpcOpenMemHandle", rc)
            opened.append(q)
            ptrs.append(q.value)
        plan.bind_external(ptrs)
        dist.barrier()
    for it in range(2):
        ins = O.seeded_inputs(d["collective"], W, nb, dt, 50 + it)
        ref = O.execute(d, ins, nb, dt)
        recv = torch.zeros(ref[rank].size, dtype=torch.uint8, device="cuda")
        plan.launch(torch.from_numpy(ins[rank]).cuda(), recv)
        torch.cuda.synchronize()
        plan.check()
        assert np.array_equal(recv.cpu().numpy(), ref[rank]), ("external", how, proto, it)
        dist.barrier()
    plan.close()
    for q in opened:
        rt.cudaIpcCloseMemHandle(q)
    dist.barrier()
    if mine.value:
        rt.cudaFree(mine)
    print("OK", rank, "external", how, proto, flush=True)
dist.destroy_process_group()
"""


@pytest.mark.parametrize("mem", ["ipc", "vmm"])
@pytest.mark.parametrize("world", [2, 4])
def test_processes_one_gpu(tmp_path, world, mem):
    """world processes, one rank each, all on cuda:0: peers' regions mapped
    through CUDA IPC handles or VMM (cuMem) POSIX fds passed over Unix sockets."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    script = tmp_path / "w.py"
    script.write_text(WORKER.format(root=ROOT, oracle=os.path.join(ROOT, "oracle"), port=port))
    env = dict(os.environ, MASTER_ADDR="127.0.0.1")
    procs = [subprocess.Popen([sys.executable, str(script), str(r), str(world), mem], stdout=subprocess.PIPE,
                              stderr=subprocess.PIPE, text=True, env=env) for r in range(world)]
    try:
        outs = [p.communicate(timeout=600) for p in procs]
    finally:
        for p in procs:
            if p.poll() is None:
                p.kill()
    for p, (o, e) in zip(procs, outs):
        assert p.returncode == 0, (o, e[-3000:])
    text = "".join(o for o, _ in outs)
    if os.environ.get("SCCL_TEST_VERBOSE"):
        print(text)
    assert text.count("OK") == (5 if world == 2 else 7) * world + 4 * world, text


FRONTIER_WORKER = r"""
import json, os, sys
sys.path[:0] = [{root!r}, {oracle!r}]
import numpy as np, torch, torch.distributed as dist
import oracle as O
from paper_2008_08708_b200 import sccl, schedules as S
rank, W = int(sys.argv[1]), int(sys.argv[2])
dist.init_process_group("gloo", init_method="tcp://127.0.0.1:{port}", rank=rank, world_size=W)
torch.cuda.set_device(0)
fdir = os.path.join({root!r}, "paper_2008_08708_b200", "frontiers")
idx = json.load(open(os.path.join(fdir, "index.json")))
import glob
gdir = os.path.join({root!r}, "tests", "golden", "schedules")
cases = []
for e in idx:
    if e["P"] == W:
        ag = open(os.path.join(fdir, e["file"])).read()
        cases.append((e["file"], ag, 8192 + 48, O.U8))
        cases.append((e["file"] + "+AR", S.allreduce_from(json.loads(ag)), 4096 * W, O.BF16))
for path in sorted(glob.glob(os.path.join(gdir, "*.json"))):  # synthesized schedules (DGX-1, AMD, ring(8) ...)
    js = open(path).read()
    d = json.loads(js)
    if d["P"] == W:
        kind = d["collective"]
        cases.append((os.path.basename(path), js, 8192 * W if kind == "alltoall" else 8192 + 48 * (kind != "allreduce"),
                      O.BF16 if kind == "allreduce" else O.U8))
n = 0
for name, js0, nb0, dt0 in cases:
    for js, nb, dt in ((js0, nb0, dt0),):
        d = json.loads(js)
        for proto in ("ll", "simple"):
            plan = sccl.Plan(js, rank, W, nb, dt, device=0, protocol=proto, timeout_ms=120000)
            plan.bind_with()
            ins = O.seeded_inputs(d["collective"], W, nb, dt, 81)
            want = O.execute(d, ins, nb, dt)[rank]
            recv = torch.full((want.size,), 0xEE, dtype=torch.uint8, device="cuda")
            plan.launch(torch.from_numpy(ins[rank]).cuda(), recv)
            torch.cuda.synchronize()
            plan.check()
            assert np.array_equal(recv.cpu().numpy(), want), (name, d["collective"], proto, rank)
            dist.barrier()
            plan.close()
            n += 1
print("OK", rank, n, flush=True)
dist.destroy_process_group()
"""


@pytest.mark.parametrize("world", [2, 4, 8])
def test_frontier_schedules_one_rank_per_process(tmp_path, world):
    """Every committed Pareto-frontier schedule of this P (ring / full /
    switch, frontiers/index.json) and the allreduce composed from it, plus
    the synthesized golden schedules of this P (DGX-1 (1,2,2) / (2,2,3) /
    (6,3,7) and their allreduces, the DGX-1 multi-hop alltoall, AMD Z52 and
    ring(8) (2,4,7)), on the
    one-rank-per-process path (IPC peers, sys-scope counters, handshake or
    parity slots), both protocols, bit-exact against the oracle on every
    rank; the processes share cuda:0."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    script = tmp_path / "f.py"
    script.write_text(FRONTIER_WORKER.format(root=ROOT, oracle=os.path.join(ROOT, "oracle"), port=port))
    env = dict(os.environ, MASTER_ADDR="127.0.0.1")
    procs = [subprocess.Popen([sys.executable, str(script), str(r), str(world)], stdout=subprocess.PIPE,
                              stderr=subprocess.PIPE, text=True, env=env) for r in range(world)]
    try:
        outs = [p.communicate(timeout=900) for p in procs]
    finally:
        for p in procs:
            if p.poll() is None:
                p.kill()
    for p, (o, e) in zip(procs, outs):
        assert p.returncode == 0, (o, e[-3000:])
    import json as _json
    idx = _json.load(open(os.path.join(ROOT, "paper_2008_08708_b200", "frontiers", "index.json")))
    golden = sum(_json.load(open(p))["P"] == world
                 for p in __import__("glob").glob(os.path.join(ROOT, "tests", "golden", "schedules", "*.json")))
    want = 2 * (2 * sum(e["P"] == world for e in idx) + golden)  # (AG + AR per frontier entry, + goldens) x 2 protocols
    counts = [int(line.split()[2]) for o, _ in outs for line in o.splitlines() if line.startswith("OK")]
    assert counts == [want] * world, (counts, want)


@pytest.mark.timeout(900)
def test_multiprocess_fuzz_four_ranks():
    """tools/fuzz_multiproc.py: 40 random valid schedules (allgather /
    reduce-scatter / allreduce, random dtype, size, protocol, CTA grid, LL
    parity on/off, counter-release mode) on the one-rank-per-process path
    with 4 processes on cuda:0, each case launched twice back to back;
    every rank bit-exact against the oracle."""
    import json as _json
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "4",
                        "--master-addr", "127.0.0.1", "--master-port", str(port),
                        os.path.join(ROOT, "tools", "fuzz_multiproc.py"), "40", "29"],
                       capture_output=True, text=True, timeout=850, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    summary = [_json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(summary) == 1 and summary[0]["cases"] == 40, r.stdout[-2000:]
    assert summary[0]["failures"] == 0, summary[0]["failed"]
