"""ctypes binding of libsccl_exec.so (the C-ABI in include/sccl_exec.h).

This is the Python face of the drop-in boundary: the reference's
``schedule.execute`` / ``cmd_exec`` become plan
creation + launch on B200.  There is no CPU or eager fallback: if the
extension is missing the import fails.
"""
from __future__ import annotations

import ctypes
import json
import os
from typing import List, Optional, Sequence

_HERE = os.path.dirname(os.path.abspath(__file__))
# SCCL_LIB: an alternative build of the same library (A/B measurements only)
LIB_PATH = os.environ.get("SCCL_LIB") or os.path.join(_HERE, "lib", "libsccl_exec.so")

OK, INVALID_ARGUMENT, CUDA_ERROR, PEER_TIMEOUT, INTERNAL = 0, 1, 4, 5, 6
U8, I32, F32, BF16, F16 = 0, 1, 2, 3, 4
SUM = 0
DTYPES = {"u8": U8, "i32": I32, "f32": F32, "bf16": BF16, "f16": F16}
ESIZE = {U8: 1, I32: 4, F32: 4, BF16: 2, F16: 2}


class SCCLError(RuntimeError):
    """Base error (maps sccl::error, /root/reference/proj/include/sccl/error.hpp:9)."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"[sccl status {code}] {msg}")
        self.code = code


class InvalidArgumentError(SCCLError, ValueError):
    """sccl::invalid_argument_error (error.hpp:14-18)."""


class PeerTimeoutError(SCCLError):
    """Watchdog fired: a peer never signalled."""


class _Opts(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int), ("nchannels", ctypes.c_int), ("chunk_groups", ctypes.c_int),
                ("tile_bytes", ctypes.c_int), ("protocol", ctypes.c_int), ("timeout_ms", ctypes.c_int64),
                ("mem_handles", ctypes.c_int), ("pull", ctypes.c_int)]


_lib = None


def lib():
    """Load the in-tree extension; raises if it was not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"libsccl_exec.so not built ({LIB_PATH}); run __graft_entry__.build() or make")
        L = ctypes.CDLL(LIB_PATH)
        c_p, c_sz = ctypes.c_void_p, ctypes.c_size_t
        L.sccl_last_error.restype = ctypes.c_char_p
        L.sccl_version.restype = ctypes.c_char_p
        for name in ("sccl_schedule_verify", "sccl_schedule_canonicalize", "sccl_schedule_invert"):
            getattr(L, name).argtypes = [ctypes.c_char_p, c_p, ctypes.POINTER(c_sz)]
        L.sccl_schedule_compose_allreduce.argtypes = [ctypes.c_char_p, ctypes.c_char_p, c_p, ctypes.POINTER(c_sz)]
        L.sccl_schedule_select.argtypes = [ctypes.POINTER(ctypes.c_char_p), ctypes.c_int, c_sz, ctypes.c_int,
                                           ctypes.c_int, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int),
                                           ctypes.POINTER(ctypes.c_double)]
        L.sccl_plan_create.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.c_int, c_sz, ctypes.c_int,
                                       ctypes.c_int, ctypes.POINTER(_Opts), ctypes.POINTER(c_p)]
        L.sccl_plan_create_loopback.argtypes = [ctypes.c_char_p, c_sz, ctypes.c_int, ctypes.c_int,
                                                ctypes.POINTER(_Opts), ctypes.POINTER(c_p)]
        L.sccl_plan_export_handles.argtypes = [c_p, c_p, ctypes.POINTER(c_sz)]
        L.sccl_plan_bind_peers.argtypes = [c_p, ctypes.POINTER(c_p), c_sz]
        L.sccl_plan_export_fd.argtypes = [c_p, ctypes.POINTER(ctypes.c_int)]
        L.sccl_plan_bind_peers_fd.argtypes = [c_p, ctypes.POINTER(c_p), c_sz, ctypes.POINTER(ctypes.c_int)]
        L.sccl_plan_recv_buffer.argtypes = [c_p, ctypes.POINTER(c_p), ctypes.POINTER(c_sz)]
        L.sccl_plan_region_bytes.argtypes = [c_p, ctypes.POINTER(c_sz)]
        L.sccl_plan_bind_peers_external.argtypes = [c_p, ctypes.POINTER(c_p)]
        L.sccl_plan_register_export.argtypes = [c_p, c_p, c_sz, c_p, ctypes.POINTER(c_sz)]
        L.sccl_plan_register_bind.argtypes = [c_p, c_p, ctypes.POINTER(c_p), c_sz]
        L.sccl_plan_deregister.argtypes = [c_p, c_p]
        L.sccl_nvls_supported.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int)]
        L.sccl_nvls_create.argtypes = [ctypes.c_int, ctypes.c_int, c_sz, ctypes.c_int, ctypes.c_int,
                                       ctypes.POINTER(c_p)]
        L.sccl_nvls_export_fd.argtypes = [c_p, ctypes.POINTER(ctypes.c_int)]
        L.sccl_nvls_join.argtypes = [c_p, ctypes.c_int]
        L.sccl_nvls_bind.argtypes = [c_p]
        L.sccl_nvls_buffer.argtypes = [c_p, ctypes.POINTER(c_p), ctypes.POINTER(c_sz)]
        L.sccl_nvls_launch.argtypes = [c_p, c_p, c_p, c_p]
        L.sccl_nvls_check.argtypes = [c_p]
        L.sccl_nvls_set_timeout.argtypes = [c_p, ctypes.c_int64]
        L.sccl_nvls_destroy.argtypes = [c_p]
        L.sccl_launch.argtypes = [c_p, c_p, c_p, c_p]
        L.sccl_launch_loopback.argtypes = [c_p, ctypes.POINTER(c_p), ctypes.POINTER(c_p), c_p]
        L.sccl_launch_loopback_copy_engine.argtypes = [c_p, ctypes.POINTER(c_p), ctypes.POINTER(c_p), c_p]
        L.sccl_plan_check.argtypes = [c_p]
        L.sccl_plan_info.argtypes = [c_p, c_p, ctypes.POINTER(c_sz)]
        L.sccl_plan_launch_count.argtypes = [c_p]
        L.sccl_plan_launch_count.restype = ctypes.c_int64
        L.sccl_plan_destroy.argtypes = [c_p]
        L.sccl_debug_interpret_loopback.argtypes = [c_p, ctypes.POINTER(c_p), ctypes.POINTER(c_p),
                                                    ctypes.c_double]
        L.sccl_debug_last_error.restype = ctypes.c_char_p
        L.sccl_debug_set_trace.argtypes = [c_p, c_p, ctypes.c_int]
        _lib = L
    return _lib


def _raise(code: int, msg: Optional[str] = None):
    if code == OK:
        return
    msg = msg if msg is not None else lib().sccl_last_error().decode()
    if code == INVALID_ARGUMENT:
        raise InvalidArgumentError(code, msg)
    if code == PEER_TIMEOUT:
        raise PeerTimeoutError(code, msg)
    raise SCCLError(code, msg)


def _string_call(fn, *args) -> str:
    n = ctypes.c_size_t(0)
    rc = fn(*args, None, ctypes.byref(n))
    if rc != OK:
        _raise(rc)
    buf = ctypes.create_string_buffer(n.value)
    rc = fn(*args, buf, ctypes.byref(n))
    _raise(rc)
    return buf.value.decode()


def _text(s) -> bytes:
    if isinstance(s, dict):
        s = json.dumps(s)
    return s.encode() if isinstance(s, str) else s


# ---------------------------------------------------------------- schedules
def canonicalize(schedule) -> str:
    """deserialize + canonical serialize."""
    return _string_call(lib().sccl_schedule_canonicalize, _text(schedule))


def verify(schedule) -> List[list]:
    """Violations [[kind, step, chunk, src, dst], ...]; [] when valid
    (SPEC.md:400-417).  Schema errors raise InvalidArgumentError."""
    L = lib()
    n = ctypes.c_size_t(1 << 20)
    buf = ctypes.create_string_buffer(n.value)
    rc = L.sccl_schedule_verify(_text(schedule), buf, ctypes.byref(n))
    if rc == OK or (rc == INVALID_ARGUMENT and buf.value.startswith(b"[")):
        return json.loads(buf.value.decode())
    _raise(rc)
    return []


def invert(schedule) -> str:
    """invert_schedule."""
    return _string_call(lib().sccl_schedule_invert, _text(schedule))


def compose_allreduce(rs, ag) -> str:
    """Allreduce = (RS, AG)."""
    return _string_call(lib().sccl_schedule_compose_allreduce, _text(rs), _text(ag))


def select(schedules: Sequence, bytes_per_rank: int, dtype: int = U8, multiprocess: bool = False):
    """Per-size algorithm + protocol choice among candidate schedules of one
    collective (e.g. a Pareto frontier) by the fitted B200 cost model
    (PAPER.md:1037).  multiprocess prices one-rank-per-GPU
    plans (system-scope constants, push lowering) instead of loopback ones.
    Returns (index, protocol name, predicted microseconds)."""
    arr = (ctypes.c_char_p * len(schedules))(*[_text(x) for x in schedules])
    idx, proto, us = ctypes.c_int(-1), ctypes.c_int(0), ctypes.c_double(0.0)
    _raise(lib().sccl_schedule_select(arr, len(schedules), bytes_per_rank, dtype, int(bool(multiprocess)),
                                      ctypes.byref(idx),
                                      ctypes.byref(proto), ctypes.byref(us)))
    return idx.value, {1: "simple", 2: "ll"}[proto.value], us.value


def version() -> str:
    return lib().sccl_version().decode()


# ---------------------------------------------------------------- plans
PROTOCOLS = {"auto": 0, "simple": 1, "ll": 2}


MEM_HANDLES = {"ipc": 0, "vmm": 1, "external": 2}


PULL = {"auto": 0, "on": 1, "off": -1}


def _opts(device: int, nchannels: int, tile_bytes: int, timeout_ms: int, chunk_groups: int = 0,
          protocol: str = "auto", mem_handles: str = "ipc", pull: str = "auto") -> _Opts:
    return _Opts(device, nchannels, chunk_groups, tile_bytes, PROTOCOLS[protocol], timeout_ms, MEM_HANDLES[mem_handles],
                 PULL[pull])


def _ptr(x) -> int:
    """device pointer of a torch tensor (or an int)"""
    if x is None:
        return 0
    if isinstance(x, int):
        return x
    return x.data_ptr()


def _stream_ptr(stream) -> int:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


class _PlanBase:
    def __init__(self):
        self._h = ctypes.c_void_p(0)

    def info(self) -> dict:
        return json.loads(_string_call(lib().sccl_plan_info, self._h))

    def check(self):
        _raise(lib().sccl_plan_check(self._h))

    def set_trace(self, buf=None, records_per_cta: int = 0):
        """Debug: event trace of the simple-protocol kernel into a zeroed
        device buffer of grid * records_per_cta * 2 u64 words (None = off)."""
        _raise(lib().sccl_debug_set_trace(self._h, _ptr(buf) if buf is not None else None, records_per_cta))

    @property
    def launch_count(self) -> int:
        return int(lib().sccl_plan_launch_count(self._h))

    def close(self):
        if self._h:
            lib().sccl_plan_destroy(self._h)
            self._h = ctypes.c_void_p(0)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class LoopbackPlan(_PlanBase):
    """Every rank of the schedule on one GPU; one launch runs them all."""

    def __init__(self, schedule, bytes_per_rank: int, dtype: int = U8, device: int = 0,
                 nchannels: int = 0, tile_bytes: int = 0, timeout_ms: int = 0, chunk_groups: int = 0,
                 protocol: str = "auto", pull: str = "auto"):
        super().__init__()
        o = _opts(device, nchannels, tile_bytes, timeout_ms, chunk_groups, protocol, pull=pull)
        rc = lib().sccl_plan_create_loopback(_text(schedule), bytes_per_rank, dtype, SUM,
                                             ctypes.byref(o), ctypes.byref(self._h))
        _raise(rc)
        meta = self.info()
        self.nranks = meta["nranks"]
        self.send_bytes = meta["program"]["send_bytes"]
        self.recv_bytes = meta["program"]["recv_bytes"]

    def launch(self, sendbufs: Sequence, recvbufs: Sequence, stream=None):
        P = self.nranks
        if len(sendbufs) < P or len(recvbufs) < P:
            raise InvalidArgumentError(INVALID_ARGUMENT, f"need {P} send and recv buffers")
        s = (ctypes.c_void_p * P)(*[_ptr(x) for x in sendbufs[:P]])
        r = (ctypes.c_void_p * P)(*[_ptr(x) for x in recvbufs[:P]])
        _raise(lib().sccl_launch_loopback(self._h, s, r, ctypes.c_void_p(_stream_ptr(stream))))

    def launch_copy_engine(self, sendbufs: Sequence, recvbufs: Sequence, stream=None):
        """Comparison backend: one cudaMemcpyAsync per send, steps in order."""
        P = self.nranks
        s = (ctypes.c_void_p * P)(*[_ptr(x) for x in sendbufs])
        r = (ctypes.c_void_p * P)(*[_ptr(x) for x in recvbufs])
        _raise(lib().sccl_launch_loopback_copy_engine(self._h, s, r, ctypes.c_void_p(_stream_ptr(stream))))

    def interpret_on_cpu(self, sendbufs: Sequence, recvbufs: Sequence, timeout_s: float = 30.0):
        """TEST HOOK (sccl_debug.h): run the lowered program on CPU threads
        over host numpy buffers.  Not an execution path of the product."""
        P = self.nranks
        s = (ctypes.c_void_p * P)(*[b.ctypes.data for b in sendbufs])
        r = (ctypes.c_void_p * P)(*[b.ctypes.data for b in recvbufs])
        rc = lib().sccl_debug_interpret_loopback(self._h, s, r, ctypes.c_double(timeout_s))
        if rc != OK:
            _raise(rc, lib().sccl_debug_last_error().decode())


class Plan(_PlanBase):
    """One rank of a one-process-per-GPU execution.  Peers' plan regions are
    mapped through CUDA IPC handles (mem_handles="ipc") or VMM cuMem
    allocations shared as POSIX file descriptors (mem_handles="vmm")."""

    def __init__(self, schedule, rank: int, nranks: int, bytes_per_rank: int, dtype: int = U8,
                 device: int = 0, nchannels: int = 0, tile_bytes: int = 0, timeout_ms: int = 0,
                 chunk_groups: int = 0, protocol: str = "auto", mem_handles: str = "ipc", pull: str = "auto"):
        super().__init__()
        self.mem_handles, self.device = mem_handles, device
        o = _opts(device, nchannels, tile_bytes, timeout_ms, chunk_groups, protocol, mem_handles, pull)
        rc = lib().sccl_plan_create(_text(schedule), rank, nranks, bytes_per_rank, dtype, SUM,
                                    ctypes.byref(o), ctypes.byref(self._h))
        _raise(rc)
        self.rank, self.nranks = rank, nranks
        meta = self.info()
        self.send_bytes = meta["program"]["send_bytes"]
        self.recv_bytes = meta["program"]["recv_bytes"]

    def export_handles(self) -> bytes:
        n = ctypes.c_size_t(0)
        lib().sccl_plan_export_handles(self._h, None, ctypes.byref(n))
        buf = ctypes.create_string_buffer(n.value)
        _raise(lib().sccl_plan_export_handles(self._h, buf, ctypes.byref(n)))
        return buf.raw[:n.value]

    def bind_peers(self, blobs: Sequence[bytes]):
        bufs = [ctypes.create_string_buffer(b, len(b)) for b in blobs]
        arr = (ctypes.c_void_p * len(bufs))(*[ctypes.addressof(b) for b in bufs])
        _raise(lib().sccl_plan_bind_peers(self._h, arr, len(blobs[0])))

    def export_fd(self) -> int:
        """VMM plans: a new POSIX fd of this rank's region (the caller closes it)."""
        fd = ctypes.c_int(-1)
        _raise(lib().sccl_plan_export_fd(self._h, ctypes.byref(fd)))
        return fd.value

    def bind_peers_fd(self, blobs: Sequence[bytes], fds: Sequence[int]):
        bufs = [ctypes.create_string_buffer(b, len(b)) for b in blobs]
        arr = (ctypes.c_void_p * len(bufs))(*[ctypes.addressof(b) for b in bufs])
        fa = (ctypes.c_int * len(fds))(*fds)
        _raise(lib().sccl_plan_bind_peers_fd(self._h, arr, len(blobs[0]), fa))

    def bind_with(self, group=None):
        """Exchange handles through torch.distributed (all_gather_object);
        VMM plans also pass their region fds over Unix sockets (SCM_RIGHTS).
        Collective, and it fails collectively: a step that raises on one rank
        raises on every rank (_collective_step), so no peer is left to time
        out in its first launch against a rank that never bound."""
        import torch.distributed as dist
        mine = _collective_step(self.export_handles, group)
        blobs: List[Optional[bytes]] = [None] * self.nranks
        dist.all_gather_object(blobs, mine, group=group)
        if self.mem_handles != "vmm":
            _collective_step(lambda: self.bind_peers(blobs), group)
            return
        fd = _collective_step(self.export_fd, group, cleanup=os.close)
        fds = _exchange_fds(self.rank, self.nranks, fd, group)
        try:
            _collective_step(lambda: self.bind_peers_fd(blobs, fds), group)
        finally:
            for r, f in enumerate(fds):
                if r != self.rank and f >= 0:
                    os.close(f)

    def register(self, buf, group=None, nbytes: Optional[int] = None):
        """Register a caller device buffer (torch tensor or pointer) as a
        zero-copy receive target: collective over torch.distributed; every
        rank registers its own buffer.  Launches with recvbuf=buf then have
        the peers write it directly.  Fails on every rank if it fails on one."""
        import torch.distributed as dist
        ptr = _ptr(buf)
        nb = nbytes if nbytes is not None else buf.numel() * buf.element_size()

        def export():
            n = ctypes.c_size_t(0)
            lib().sccl_plan_register_export(self._h, ctypes.c_void_p(ptr), nb, None, ctypes.byref(n))
            mine = ctypes.create_string_buffer(n.value)
            _raise(lib().sccl_plan_register_export(self._h, ctypes.c_void_p(ptr), nb, mine, ctypes.byref(n)))
            return mine.raw[:n.value]
        mine = _collective_step(export, group)
        blobs: List[Optional[bytes]] = [None] * self.nranks
        dist.all_gather_object(blobs, mine, group=group)
        bufs = [ctypes.create_string_buffer(b, len(b)) for b in blobs]
        arr = (ctypes.c_void_p * len(bufs))(*[ctypes.addressof(b) for b in bufs])
        _collective_step(lambda: _raise(lib().sccl_plan_register_bind(self._h, ctypes.c_void_p(ptr), arr,
                                                                       len(blobs[0]))), group)

    def deregister(self, buf):
        _raise(lib().sccl_plan_deregister(self._h, ctypes.c_void_p(_ptr(buf))))

    def region_bytes(self) -> int:
        n = ctypes.c_size_t(0)
        _raise(lib().sccl_plan_region_bytes(self._h, ctypes.byref(n)))
        return n.value

    def bind_external(self, regions: Sequence[int]):
        """Bind to caller-provided regions (mem_handles="external"):
        regions[r] = rank r's region as mapped in this process."""
        arr = (ctypes.c_void_p * len(regions))(*regions)
        _raise(lib().sccl_plan_bind_peers_external(self._h, arr))

    def bind_symmetric_memory(self, group=None):
        """mem_handles="external" through torch symmetric memory (SURVEY.md
        8(f) f4, a production integration path): the plan region is a
        symm_mem.empty tensor, rendezvous gives every peer's mapping of its
        counterpart, and the plan runs on those (no IPC / fd exchange of our
        own).  Collective; checks that every rank lowered the same plan."""
        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm_mem
        info = self.info()
        key = (info["program"]["fingerprint"], info["nchannels"], info["tile_bytes"], info["protocol"],
               self.region_bytes())
        keys: List[Optional[tuple]] = [None] * self.nranks
        dist.all_gather_object(keys, key, group=group)
        if any(k != key for k in keys):
            raise InvalidArgumentError(INVALID_ARGUMENT, f"ranks lowered different plans: {keys}")
        t = symm_mem.empty(self.region_bytes(), dtype=torch.uint8, device=torch.device("cuda", self.device))
        hdl = symm_mem.rendezvous(t, group if group is not None else dist.group.WORLD)
        _collective_step(lambda: self.bind_external(list(hdl.buffer_ptrs)), group)
        dist.barrier(group=group)  # every region zeroed before any rank's first launch
        self._symm = (t, hdl)

    def recv_buffer(self):
        p = ctypes.c_void_p(0)
        n = ctypes.c_size_t(0)
        _raise(lib().sccl_plan_recv_buffer(self._h, ctypes.byref(p), ctypes.byref(n)))
        return p.value, n.value

    def launch(self, sendbuf, recvbuf=None, stream=None):
        _raise(lib().sccl_launch(self._h, ctypes.c_void_p(_ptr(sendbuf)), ctypes.c_void_p(_ptr(recvbuf)),
                                 ctypes.c_void_p(_stream_ptr(stream))))


def _collective_step(fn, group=None, cleanup=None):
    """One local step of a collective setup (export, bind, join ...), run on
    every rank, then agreed: if it raised on any rank, it raises on every rank
    -- the first failing rank's status, every failing rank's message -- so no
    rank goes on into a later collective (a barrier, a fd exchange, a launch
    whose peers wait for its entry flag) that a failed peer never reaches.
    cleanup(result) releases this rank's result when another rank failed."""
    import torch.distributed as dist
    res, err = None, None
    try:
        res = fn()
    except SCCLError as e:
        err = (e.code, str(e))
    except Exception as e:  # noqa: BLE001 -- reported on every rank below
        err = (INTERNAL, f"{type(e).__name__}: {e}")
    errs: List[Optional[tuple]] = [None] * dist.get_world_size(group)
    dist.all_gather_object(errs, err, group=group)
    bad = [(r, e) for r, e in enumerate(errs) if e is not None]
    if bad:
        if err is None and cleanup is not None and res is not None:
            cleanup(res)
        _raise(bad[0][1][0], f"collective step failed on rank(s) {[r for r, _ in bad]}: " +
               "; ".join(f"rank {r}: {e[1]}" for r, e in bad))
    return res


def _exchange_fds(rank: int, nranks: int, my_fd: int, group=None) -> List[int]:
    """All-to-all of one file descriptor per rank over Linux abstract Unix
    sockets (SCM_RIGHTS); the socket names travel through torch.distributed.
    Returns fds[r] = a local fd for rank r's descriptor (fds[rank] = -1).
    Consumes (closes) my_fd."""
    import socket
    import threading
    import uuid
    import torch.distributed as dist
    name = f"\0sccl-{uuid.uuid4().hex}-{rank}"
    srv = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
    srv.bind(name)
    srv.listen(nranks)
    names: List[Optional[str]] = [None] * nranks
    dist.all_gather_object(names, name, group=group)
    fds = [-1] * nranks

    def send_all():
        for r in range(nranks):
            if r == rank:
                continue
            c = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
            c.connect(names[r])
            socket.send_fds(c, [rank.to_bytes(4, "little")], [my_fd])
            c.close()

    t = threading.Thread(target=send_all)
    t.start()
    try:
        for _ in range(nranks - 1):
            conn, _ = srv.accept()
            msg, got, _, _ = socket.recv_fds(conn, 4, 1)
            fds[int.from_bytes(msg, "little")] = got[0]
            conn.close()
    finally:
        t.join()
        srv.close()
        os.close(my_fd)
    dist.barrier(group=group)
    return fds


class AutoLoopbackPlan:
    """Per-size algorithm switching over a set of synthesized schedules of one
    collective (e.g. a Pareto frontier; "automatically switch
    between multiple implementations"): each new per-rank byte count picks
    its schedule and protocol with `select` (the fitted B200 cost model) and
    caches the plan; launches reuse it."""

    def __init__(self, schedules: Sequence, dtype: int = U8, device: int = 0, max_plans: int = 16):
        self.schedules = [_text(s).decode() for s in schedules]
        self.dtype, self.device, self.max_plans = dtype, device, max_plans
        self._plans = {}  # bytes_per_rank -> (schedule index, protocol, LoopbackPlan)
        self.discovery = None

    @classmethod
    def from_machine(cls, collective: str = "allgather", P: int = 8, dtype: int = U8, device: int = 0,
                     max_plans: int = 16):
        """Candidates from topology discovery (frontier.for_this_machine):
        on one GPU, every committed Pareto frontier for P ranks."""
        from . import frontier
        info, scheds = frontier.for_this_machine(collective, P)
        self = cls(scheds, dtype, device, max_plans)
        self.discovery = info
        return self

    def plan_for(self, bytes_per_rank: int):
        if bytes_per_rank not in self._plans:
            if len(self._plans) >= self.max_plans:  # evict the oldest
                oldest = next(iter(self._plans))
                self._plans.pop(oldest)[2].close()
            i, proto, _ = select(self.schedules, bytes_per_rank, self.dtype)
            self._plans[bytes_per_rank] = (i, proto, LoopbackPlan(self.schedules[i], bytes_per_rank, self.dtype,
                                                                  device=self.device, protocol=proto))
        return self._plans[bytes_per_rank]

    def launch(self, sendbufs: Sequence, recvbufs: Sequence, bytes_per_rank: int, stream=None):
        i, proto, plan = self.plan_for(bytes_per_rank)
        plan.launch(sendbufs, recvbufs, stream)
        return i, proto

    def check(self):
        for _, _, plan in self._plans.values():
            plan.check()

    def close(self):
        for _, _, plan in self._plans.values():
            plan.close()
        self._plans.clear()


class AutoPlan:
    """One rank of a one-process-per-GPU execution with per-size algorithm
    switching: each new per-rank byte count picks its
    schedule and protocol with `select(..., multiprocess=True)` (the
    system-scope cost model), creates that rank's Plan and binds it to the
    peers (collective: every rank must launch the same sizes in the same
    order, as SPMD code does)."""

    def __init__(self, schedules: Sequence, rank: int, nranks: int, dtype: int = U8, device: int = 0,
                 group=None, mem_handles: str = "ipc", max_plans: int = 16):
        self.schedules = [_text(s).decode() for s in schedules]
        self.rank, self.nranks, self.dtype, self.device = rank, nranks, dtype, device
        self.group, self.mem_handles, self.max_plans = group, mem_handles, max_plans
        self._plans = {}
        self.discovery = None

    @classmethod
    def from_machine(cls, collective: str, rank: int, nranks: int, dtype: int = U8, device: int = 0,
                     group=None, mem_handles: str = "ipc"):
        """Candidates for the discovered target (switch:N on an NVSwitch
        box: the switch(N) and full(N) frontiers)."""
        from . import frontier
        from . import topology
        info = topology.discover()
        target = info["target"] if info["target"].split(":")[0] in ("switch", "full") else f"full:{nranks}"
        self = cls(frontier.candidates(collective, target, nranks), rank, nranks, dtype, device, group, mem_handles)
        self.discovery = dict(info, used_target=target)
        return self

    def plan_for(self, bytes_per_rank: int):
        if bytes_per_rank not in self._plans:
            if len(self._plans) >= self.max_plans:
                self._plans.pop(next(iter(self._plans)))[2].close()
            i, proto, _ = select(self.schedules, bytes_per_rank, self.dtype, multiprocess=True)
            plan = Plan(self.schedules[i], self.rank, self.nranks, bytes_per_rank, self.dtype, device=self.device,
                        protocol=proto, mem_handles=self.mem_handles)
            plan.bind_with(self.group)
            self._plans[bytes_per_rank] = (i, proto, plan)
        return self._plans[bytes_per_rank]

    def launch(self, sendbuf, recvbuf, bytes_per_rank: int, stream=None):
        i, proto, plan = self.plan_for(bytes_per_rank)
        plan.launch(sendbuf, recvbuf, stream)
        return i, proto

    def check(self):
        for _, _, plan in self._plans.values():
            plan.check()

    def close(self):
        for _, _, plan in self._plans.values():
            plan.close()
        self._plans.clear()


def nvls_supported(device: int = 0, nranks: int = 1) -> bool:
    """The device can form a multicast team of nranks GPUs (the attribute
    plus a trial cuMulticastCreate)."""
    v = ctypes.c_int(0)
    _raise(lib().sccl_nvls_supported(device, nranks, ctypes.byref(v)))
    return bool(v.value)


def _share_fd_from_root(rank: int, nranks: int, fd: int, group=None) -> int:
    """Rank 0's file descriptor to every other rank (SCM_RIGHTS over Linux
    abstract Unix sockets; the socket names travel through torch.distributed).
    Returns the local fd (rank 0: -1, and its fd is closed)."""
    import socket
    import uuid
    import torch.distributed as dist
    name = f"\0sccl-nvls-{uuid.uuid4().hex}-{rank}"
    srv = None
    if rank != 0:
        srv = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
        srv.bind(name)
        srv.listen(1)
    names: List[Optional[str]] = [None] * nranks
    dist.all_gather_object(names, name, group=group)
    got = -1
    if rank == 0:
        for r in range(1, nranks):
            c = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
            c.connect(names[r])
            socket.send_fds(c, [b"fd"], [fd])
            c.close()
        os.close(fd)
    else:
        conn, _ = srv.accept()
        _, fds, _, _ = socket.recv_fds(conn, 2, 1)
        got = fds[0]
        conn.close()
        srv.close()
    dist.barrier(group=group)
    return got


class NvlsAllreduce:
    """NVLS allreduce (SURVEY.md 8(f) f4 comparison backend): every rank's
    buffer bound to one CUDA multicast object, rank r reduces slice r inside
    the NVSwitch (multimem.ld_reduce / multimem.st).  One rank per GPU;
    nranks = 1 needs no process group (a one-device multicast team)."""

    def __init__(self, rank: int, nranks: int, nbytes: int, dtype: int = BF16, device: int = 0, group=None,
                 timeout_ms: int = 0):
        """timeout_ms: barrier watchdog (0 = 600 s, < 0 = off).  Collective for nranks > 1, and it fails collectively: every step
        (create, rank 0's export, join, bind) is agreed across the ranks
        (_collective_step), so a multicast team that cannot form raises on
        every rank instead of leaving peers in a barrier."""
        self._h = ctypes.c_void_p(0)
        self.rank, self.nranks, self.nbytes = rank, nranks, nbytes
        multi = nranks > 1
        step = (lambda fn, **kw: _collective_step(fn, group, **kw)) if multi else (lambda fn, **kw: fn())
        step(lambda: _raise(lib().sccl_nvls_create(rank, nranks, nbytes, dtype, device, ctypes.byref(self._h))))
        _raise(lib().sccl_nvls_set_timeout(self._h, timeout_ms))
        fd = -1
        if multi:
            import torch.distributed as dist

            def export():
                if rank != 0:
                    return -1
                f = ctypes.c_int(-1)
                _raise(lib().sccl_nvls_export_fd(self._h, ctypes.byref(f)))
                return f.value
            fd = step(export, cleanup=lambda f: os.close(f) if f >= 0 else None)
            fd = _share_fd_from_root(rank, nranks, fd, group)

        def join():
            try:
                _raise(lib().sccl_nvls_join(self._h, fd))
            finally:
                if fd >= 0:
                    os.close(fd)
        step(join)
        if multi:
            dist.barrier(group=group)  # every device is in the team before anyone binds
        step(lambda: _raise(lib().sccl_nvls_bind(self._h)))
        if multi:
            dist.barrier(group=group)

    def buffer(self):
        p, n = ctypes.c_void_p(0), ctypes.c_size_t(0)
        _raise(lib().sccl_nvls_buffer(self._h, ctypes.byref(p), ctypes.byref(n)))
        return p.value, n.value

    def launch(self, sendbuf=None, recvbuf=None, stream=None):
        _raise(lib().sccl_nvls_launch(self._h, ctypes.c_void_p(_ptr(sendbuf)), ctypes.c_void_p(_ptr(recvbuf)),
                                      ctypes.c_void_p(_stream_ptr(stream))))

    def check(self):
        _raise(lib().sccl_nvls_check(self._h))

    def close(self):
        if self._h:
            lib().sccl_nvls_destroy(self._h)
            self._h = ctypes.c_void_p(0)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
