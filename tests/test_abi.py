"""The C-ABI boundary: libsccl_exec.so loads, exports every symbol the
headers declare, maps errors to the documented status codes, and the
multi-process handle exchange works across processes (gloo, world 2)."""
import ctypes
import os
import re
import subprocess

import pytest

from paper_2008_08708_b200 import sccl
from paper_2008_08708_b200 import schedules as S

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared(header):
    text = open(os.path.join(ROOT, "include", header)).read()
    return sorted(set(re.findall(r"\b(sccl_[a-z_]+)\s*\(", text)) - {"sccl_plan_opts"})


@pytest.mark.parametrize("header", ["sccl_exec.h", "sccl_debug.h"])
def test_library_exports_declared_symbols(header):
    names = _declared(header)
    assert len(names) >= 2
    out = subprocess.run(["nm", "-D", "--defined-only", sccl.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (sccl_\w+)", out))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    L = sccl.lib()
    for n in names:
        assert getattr(L, n) is not None


def test_kernels_are_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", sccl.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version_and_last_error():
    assert "sm_100a" in sccl.version()
    with pytest.raises(sccl.InvalidArgumentError) as e:
        sccl.canonicalize('{"collective":"nope"}')
    assert e.value.code == sccl.INVALID_ARGUMENT


def test_host_only_plan_cannot_launch():
    js = S.to_json(S.one_shot_allgather(4))
    p = sccl.LoopbackPlan(js, 4096, sccl.U8, device=-1)
    with pytest.raises(sccl.InvalidArgumentError, match="host-only"):
        p.launch([0] * 4, [0] * 4, stream=0)
    q = sccl.Plan(js, 1, 4, 4096, sccl.U8, device=-1)
    with pytest.raises(sccl.InvalidArgumentError, match="host-only|not bound"):
        q.launch(0, 0, stream=0)


def test_bad_arguments():
    js = S.to_json(S.one_shot_allgather(4))
    with pytest.raises(sccl.InvalidArgumentError, match="nranks"):
        sccl.Plan(js, 0, 8, 4096, sccl.U8, device=-1)
    with pytest.raises(sccl.InvalidArgumentError, match="rank"):
        sccl.Plan(js, 4, 4, 4096, sccl.U8, device=-1)
    with pytest.raises(sccl.InvalidArgumentError, match="multiple of the element size"):
        sccl.LoopbackPlan(S.allreduce_from(S.one_shot_allgather(4)), 4098, sccl.F32, device=-1)
    with pytest.raises(sccl.InvalidArgumentError, match="tile"):
        sccl.LoopbackPlan(js, 4096, sccl.U8, device=-1, tile_bytes=100)
    with pytest.raises(sccl.InvalidArgumentError, match="tile"):
        sccl.LoopbackPlan(js, 4096, sccl.U8, device=-1, tile_bytes=131072)


def test_blob_exchange_single_process():
    js = S.to_json(S.hamiltonian_allgather(8))
    plans = [sccl.Plan(js, r, 8, 1 << 16, sccl.U8, device=-1) for r in range(8)]
    blobs = [p.export_handles() for p in plans]
    for p in plans:
        p.bind_peers(blobs)
    with pytest.raises(sccl.InvalidArgumentError, match="already bound"):
        plans[0].bind_peers(blobs)
    other = sccl.Plan(js, 3, 8, 1 << 17, sccl.U8, device=-1)  # different size -> different program
    fresh = sccl.Plan(js, 0, 8, 1 << 16, sccl.U8, device=-1)
    bad = list(blobs)
    bad[3] = other.export_handles()
    with pytest.raises(sccl.InvalidArgumentError, match="fingerprint"):
        fresh.bind_peers(bad)
    bad = list(blobs)
    bad[2], bad[4] = bad[4], bad[2]
    with pytest.raises(sccl.InvalidArgumentError, match="rank"):
        fresh.bind_peers(bad)


_WORKER = r"""
import os, sys
sys.path.insert(0, {root!r})
import torch.distributed as dist
from paper_2008_08708_b200 import sccl, schedules as S
dist.init_process_group("gloo", init_method="tcp://127.0.0.1:{port}", rank=int(sys.argv[1]), world_size=2)
r = dist.get_rank()
js = S.to_json(S.one_shot_allgather(2))
nbytes = 4096 if (r == 0 or sys.argv[2] == "same") else 8192
p = sccl.Plan(js, r, 2, nbytes, sccl.U8, device=-1)
try:
    p.bind_with()
    print("BOUND", r, p.info()["program"]["fingerprint"], flush=True)
except sccl.InvalidArgumentError as e:
    print("MISMATCH", r, str(e)[:60], flush=True)
dist.destroy_process_group()
"""


@pytest.mark.parametrize("mode", ["same", "differ"])
def test_gloo_two_process_handle_exchange(tmp_path, mode):
    """world_size-2 gloo: each rank lowers the schedule, exchanges its blob
    through torch.distributed and binds; mismatched programs are refused."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    script = tmp_path / "w.py"
    script.write_text(_WORKER.format(root=ROOT, port=port))
    env = dict(os.environ, MASTER_ADDR="127.0.0.1")
    procs = [subprocess.Popen(["python", str(script), str(r), mode], stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                              text=True, env=env) for r in range(2)]
    outs = [p.communicate(timeout=120) for p in procs]
    for p, (o, e) in zip(procs, outs):
        assert p.returncode == 0, e
    text = "".join(o for o, _ in outs)
    if mode == "same":
        assert text.count("BOUND") == 2
        fps = {line.split()[2] for line in text.splitlines() if line.startswith("BOUND")}
        assert len(fps) == 1
    else:
        assert text.count("MISMATCH") == 2


_FAIL_WORKER = r"""
import sys
sys.path.insert(0, {root!r})
import torch.distributed as dist
from paper_2008_08708_b200 import sccl, schedules as S
dist.init_process_group("gloo", init_method="tcp://127.0.0.1:{port}", rank=int(sys.argv[1]), world_size=2)
r = dist.get_rank()
p = sccl.Plan(S.to_json(S.one_shot_allgather(2)), r, 2, 4096, sccl.U8, device=-1)
if r == 1:  # only rank 1's local bind fails (e.g. a peer mapping the driver refuses)
    def bad(blobs):
        raise sccl.SCCLError(sccl.CUDA_ERROR, "injected cudaIpcOpenMemHandle failure")
    p.bind_peers = bad
try:
    p.bind_with()
    print("BOUND", r, flush=True)
except sccl.SCCLError as e:
    print("FAILED", r, e.code, "rank 1: [sccl status 4] injected" in str(e), flush=True)
dist.barrier()  # both ranks reach the next collective: nobody was left waiting
print("NEXT", r, flush=True)
dist.destroy_process_group()
"""


def test_bind_fails_on_every_rank_when_one_rank_fails(tmp_path):
    """bind_with is collective and fails collectively (_collective_step):
    one rank's failed local bind raises on both ranks of a world-size-2 gloo
    job, with the failing rank's status and message, and both go on to the
    next collective instead of one of them waiting on a peer that gave up."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    script = tmp_path / "fail.py"
    script.write_text(_FAIL_WORKER.format(root=ROOT, port=port))
    env = dict(os.environ, MASTER_ADDR="127.0.0.1")
    procs = [subprocess.Popen(["python", str(script), str(r)], stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                              text=True, env=env) for r in range(2)]
    outs = [p.communicate(timeout=120) for p in procs]
    for p, (o, e) in zip(procs, outs):
        assert p.returncode == 0, e
    text = "".join(o for o, _ in outs)
    assert "FAILED 0 4 True" in text and "FAILED 1 4 True" in text, text
    assert text.count("NEXT") == 2 and "BOUND" not in text


_FD_WORKER = r"""
import os, sys
sys.path.insert(0, {root!r})
import torch.distributed as dist
from paper_2008_08708_b200 import sccl
dist.init_process_group("gloo", init_method="tcp://127.0.0.1:{port}", rank=int(sys.argv[1]), world_size=3)
r = dist.get_rank()
fd0 = os.memfd_create("sccl-test")  # stands in for a cuMem region fd: any descriptor travels the same way
os.write(fd0, b"rank%d" % r)
fds = sccl._exchange_fds(r, 3, fd0)
for q, fd in enumerate(fds):
    if q == r:
        assert fd == -1
    else:
        assert os.pread(fd, 16, 0) == b"rank%d" % q, (r, q)
        os.close(fd)
print("FDS_OK", r, flush=True)
dist.destroy_process_group()
"""


def test_fd_exchange_three_processes(tmp_path):
    """VMM handle path, host side: every rank's file descriptor reaches every
    other rank over abstract Unix sockets (SCM_RIGHTS), world size 3, gloo."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    script = tmp_path / "fd.py"
    script.write_text(_FD_WORKER.format(root=ROOT, port=port))
    env = dict(os.environ, MASTER_ADDR="127.0.0.1")
    procs = [subprocess.Popen(["python", str(script), str(r)], stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                              text=True, env=env) for r in range(3)]
    outs = [p.communicate(timeout=120) for p in procs]
    for p, (o, e) in zip(procs, outs):
        assert p.returncode == 0, e
    assert "".join(o for o, _ in outs).count("FDS_OK") == 3


def test_vmm_plan_host_only_errors():
    js = S.to_json(S.one_shot_allgather(2))
    p = sccl.Plan(js, 0, 2, 4096, sccl.U8, device=-1, mem_handles="vmm")
    with pytest.raises(sccl.InvalidArgumentError, match="host-only"):
        p.export_fd()
    ipc = sccl.Plan(js, 0, 2, 4096, sccl.U8, device=-1)
    with pytest.raises(sccl.InvalidArgumentError, match="VMM"):
        ipc.export_fd()
    blobs = [p.export_handles(), sccl.Plan(js, 1, 2, 4096, sccl.U8, device=-1, mem_handles="vmm").export_handles()]
    with pytest.raises(sccl.InvalidArgumentError, match="bind_peers_fd"):
        p.bind_peers(blobs)


def test_register_buffer_host_only():
    """sccl_plan_register_export / _bind on host-only plans (no CUDA): the
    size and alignment checks, the blob exchange, double registration."""
    import ctypes
    js = S.allreduce_from(S.one_shot_allgather(2))
    plans = [sccl.Plan(js, r, 2, 4096, sccl.F32, device=-1) for r in range(2)]
    blobs = [p.export_handles() for p in plans]
    for p in plans:
        p.bind_peers(blobs)
    L = sccl.lib()
    bufs = [ctypes.create_string_buffer(4096 + 16) for _ in range(2)]
    ptrs = [(ctypes.addressof(b) + 15) // 16 * 16 for b in bufs]
    n = ctypes.c_size_t(0)
    assert L.sccl_plan_register_export(plans[0]._h, ctypes.c_void_p(ptrs[0]), 4096, None, ctypes.byref(n)) == 0
    regs = []
    for p, ptr in zip(plans, ptrs):
        blob = ctypes.create_string_buffer(n.value)
        m = ctypes.c_size_t(n.value)
        assert L.sccl_plan_register_export(p._h, ctypes.c_void_p(ptr), 4096, blob, ctypes.byref(m)) == 0
        regs.append(blob)
        small = ctypes.create_string_buffer(n.value)
        assert L.sccl_plan_register_export(p._h, ctypes.c_void_p(ptr), 1024, small,
                                           ctypes.byref(ctypes.c_size_t(n.value))) == sccl.INVALID_ARGUMENT
    arr = (ctypes.c_void_p * 2)(*[ctypes.addressof(b) for b in regs])
    for p, ptr in zip(plans, ptrs):
        assert L.sccl_plan_register_bind(p._h, ctypes.c_void_p(ptr), arr, n.value) == 0
        assert L.sccl_plan_register_bind(p._h, ctypes.c_void_p(ptr), arr, n.value) == sccl.INVALID_ARGUMENT
        assert L.sccl_plan_deregister(p._h, ctypes.c_void_p(ptr)) == 0
        assert L.sccl_plan_deregister(p._h, ctypes.c_void_p(ptr)) == sccl.INVALID_ARGUMENT


def test_bind_rejects_dtype_mismatch():
    """Ranks that lowered the same program for different element formats
    (bf16 vs f16: same element size, same fingerprint) must not bind."""
    js = S.allreduce_from(S.one_shot_allgather(2))
    a = sccl.Plan(js, 0, 2, 4096, sccl.BF16, device=-1)
    b = sccl.Plan(js, 1, 2, 4096, sccl.F16, device=-1)
    with pytest.raises(sccl.InvalidArgumentError, match="dtype"):
        a.bind_peers([a.export_handles(), b.export_handles()])
