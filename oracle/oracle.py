"""CPU oracle for the synthesized-collective executor -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this module.  It is the checker, never
the thing measured or shipped; the product package never imports it.

What it restates (all citations into /root/reference):
  * topology builders        SPEC.md:36-71   (ring, full, dgx1, amd-z52) plus
                             the NVSwitch egress/ingress model
  * collective relations     SPEC.md:129-182 (All/Root/Scattered/Transpose,
                             to_global, make_spec; chunk id i*P+n SPEC.md:191)
  * schedule verify          SPEC.md:400-408        -> C: oracle_verify
  * verify_combining         SPEC.md:409-417        -> C: oracle_verify_combining
  * execute                  SPEC.md:418-426,442-447 -> C: oracle_execute
  * composition AR = (RS,AG) SPEC.md:347-355
and the buffer layout of SURVEY.md Appendix C (chunk id -> byte offset) with
the 16-byte-aligned chunk split of Appendix A8, which the GPU executor shares
by definition.

Parity status: the reference ships no executor; this
oracle is pinned by the SPEC's textual known-answer examples, committed as
tests/golden/*.json by tools/make_golden.py, and by a second, pure-Python
restatement (``execute_py``) used on small cases.
"""
from __future__ import annotations

import ctypes
import hashlib
import json
import os
import subprocess
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libsccl_oracle.so")

U8, I32, F32, BF16, F16 = 0, 1, 2, 3, 4
ESIZE = {U8: 1, I32: 4, F32: 4, BF16: 2, F16: 2}
NP_DTYPE = {U8: np.uint8, I32: np.int32, F32: np.float32, BF16: np.uint16, F16: np.float16}
DTYPE_NAMES = {"u8": U8, "i32": I32, "f32": F32, "bf16": BF16, "f16": F16}

COMBINING = {"reduce", "reducescatter", "allreduce"}
ROOTED = {"broadcast", "reduce", "gather", "scatter"}

V_NAMES = {1: "schema", 2: "edge", 3: "unavailable", 4: "bandwidth", 5: "post",
           6: "duplicate", 7: "multiplicity"}


# --------------------------------------------------------------------------
# build / load the C library
# --------------------------------------------------------------------------
def build(force: bool = False) -> str:
    src = os.path.join(HERE, "sccl_oracle.c")
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["make", "-s", "-C", HERE])
    return LIB_PATH


_lib = None


class _Viol(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("step", ctypes.c_int32), ("chunk", ctypes.c_int32),
                ("src", ctypes.c_int32), ("dst", ctypes.c_int32)]


class _Topo(ctypes.Structure):
    _fields_ = [("P", ctypes.c_int32), ("ncons", ctypes.c_int32),
                ("cons_off", ctypes.c_void_p), ("cons_edges", ctypes.c_void_p),
                ("cons_bound", ctypes.c_void_p)]


class _Sched(ctypes.Structure):
    _fields_ = [("G", ctypes.c_int32), ("S", ctypes.c_int32), ("rounds", ctypes.c_void_p),
                ("nsends", ctypes.c_int32), ("sends", ctypes.c_void_p)]


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB_PATH)
        L.oracle_verify.restype = ctypes.c_int
        L.oracle_verify_combining.restype = ctypes.c_int
        L.oracle_execute.restype = ctypes.c_int
        L.oracle_memcpy_bw.restype = ctypes.c_double
        L.oracle_memcpy_bw.argtypes = [ctypes.c_int64, ctypes.c_int, ctypes.c_int]
        _lib = L
    return _lib


# --------------------------------------------------------------------------
# topology
# --------------------------------------------------------------------------
def _pairs_topo(name: str, P: int, edges_bounds) -> dict:
    return {"name": name, "P": P,
            "constraints": [{"edges": [list(e)], "bound": b} for e, b in edges_bounds]}


def build_ring(P: int, bw: int = 1) -> dict:
    if P < 2:
        raise ValueError("ring needs P >= 2")
    eb = []
    seen = set()
    for i in range(P):
        for e in ((i, (i + 1) % P), ((i + 1) % P, i)):
            if e not in seen:
                seen.add(e)
                eb.append((e, bw))
    return _pairs_topo(f"ring:{P}", P, eb)


def build_full(P: int, bw: int = 1) -> dict:
    return _pairs_topo(f"full:{P}", P, [((a, b), bw) for a in range(P) for b in range(P) if a != b])


def build_dgx1() -> dict:
    """two Hamiltonian cycles, double- and single-NVLink."""
    eb = {}
    for cyc, bw in (((0, 1, 4, 5, 6, 7, 2, 3), 2), ((0, 2, 1, 3, 6, 4, 7, 5), 1)):
        for i in range(8):
            a, b = cyc[i], cyc[(i + 1) % 8]
            eb[(a, b)] = eb.get((a, b), 0) + bw
            eb[(b, a)] = eb.get((b, a), 0) + bw
    return _pairs_topo("dgx1", 8, sorted(eb.items()))


def build_amd_z52() -> dict:
    t = build_ring(8, 1)
    t["name"] = "amd-z52"
    return t


def build_switch(P: int, bw: int = 1) -> dict:
    """NVSwitch box: every pair linked, each GPU sends <= bw and receives <= bw
    chunks per round (grouped constraints)."""
    cons = []
    for n in range(P):
        cons.append({"edges": [[n, d] for d in range(P) if d != n], "bound": bw})
    for n in range(P):
        cons.append({"edges": [[s, n] for s in range(P) if s != n], "bound": bw})
    return {"name": f"switch:{P}", "P": P, "constraints": cons}


def topology_by_name(name: str) -> dict:
    if name == "dgx1":
        return build_dgx1()
    if name == "amd-z52":
        return build_amd_z52()
    kind, _, arg = name.partition(":")
    P = int(arg)
    return {"ring": build_ring, "full": build_full, "switch": build_switch}[kind](P)


def topology_hash(t: dict) -> str:
    """FNV-1a 64 over the canonical constraint text."""
    cons = sorted((sorted(tuple(e) for e in c["edges"]), c["bound"]) for c in t["constraints"])
    text = f"{t['P']}|" + ";".join(
        f"{b}:" + ",".join(f"{a}>{d}" for a, d in edges) for edges, b in cons)
    h = 0xcbf29ce484222325
    for ch in text.encode():
        h ^= ch
        h = (h * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return f"{h:016x}"


# --------------------------------------------------------------------------
# collectives
# --------------------------------------------------------------------------
def relation(kind: str, G: int, P: int, root: int = 0) -> np.ndarray:
    """G x P boolean matrix."""
    m = np.zeros((G, P), dtype=np.uint8)
    if kind == "all":
        m[:] = 1
    elif kind == "root":
        m[:, root] = 1
    elif kind == "scattered":
        assert G % P == 0
        m[np.arange(G), np.arange(G) % P] = 1
    elif kind == "transpose":
        assert G % (P * P) == 0
        m[np.arange(G), (np.arange(G) // P) % P] = 1
    else:
        raise ValueError(kind)
    return m


def to_global(kind: str, C: int, P: int) -> int:
    if kind in ("broadcast", "reduce"):
        return C
    if kind == "alltoall" and C % P:
        raise ValueError("alltoall needs C mod P == 0")
    return P * C


# Table 2: (pre, post) of the non-combining collective, or
# of the non-combining dual for combining ones.
_SPEC = {
    "gather": ("scattered", "root"), "allgather": ("scattered", "all"),
    "alltoall": ("scattered", "transpose"), "broadcast": ("root", "all"),
    "scatter": ("root", "scattered"),
    "reduce": ("root", "all"), "reducescatter": ("scattered", "all"),
}


def pre_post(kind: str, G: int, P: int, root: int = 0):
    """Non-combining: (pre, post).  Combining: (contrib, dest) =
    (dual post, dual pre) -- the inversion of SPEC.md:338-355."""
    a, b = _SPEC[kind]
    pa, pb = relation(a, G, P, root), relation(b, G, P, root)
    if kind in COMBINING:
        return pb, pa
    return pa, pb


# --------------------------------------------------------------------------
# layout (split rule Appendix A8)
# --------------------------------------------------------------------------
def split(L: int, K: int, i: int) -> Tuple[int, int]:
    """Part i of K of an L-byte range: 16-byte aligned starts, remainder in
    the last part.  Returns (offset, length)."""
    U = L // 16
    lo = (i * U // K) * 16
    hi = L if i == K - 1 else ((i + 1) * U // K) * 16
    return lo, hi - lo


def buffer_sizes(kind: str, P: int, nbytes: int) -> Tuple[int, int]:
    """(send bytes, recv bytes) per rank for the per-rank size argument."""
    if kind == "allgather":
        return nbytes, P * nbytes
    if kind == "reducescatter":
        return P * nbytes, nbytes
    if kind == "gather":
        return nbytes, P * nbytes
    if kind == "scatter":
        return P * nbytes, nbytes
    return nbytes, nbytes


def chunk_geometry(kind: str, P: int, C: int, nbytes: int, G: int):
    """For every chunk: (length, input offset, output offset).  Offsets are
    the same on every rank that holds the chunk in that buffer."""
    geo = []
    for c in range(G):
        if kind in ("allgather", "gather"):
            n, i = c % P, c // P
            off, ln = split(nbytes, C, i)
            geo.append((ln, off, n * nbytes + off))
        elif kind in ("reducescatter", "scatter"):
            n, i = c % P, c // P
            off, ln = split(nbytes, C, i)
            geo.append((ln, n * nbytes + off, off))
        elif kind in ("broadcast", "reduce"):
            off, ln = split(nbytes, C, c)
            geo.append((ln, off, off))
        elif kind == "allreduce":
            n, i = c % P, c // P
            so, sl = split(nbytes, P, n)
            off, ln = split(sl, G // P, i)
            geo.append((ln, so + off, so + off))
        elif kind == "alltoall":
            assert nbytes % P == 0
            seg = nbytes // P
            src, dst, j = c % P, (c // P) % P, c // (P * P)
            off, ln = split(seg, C // P, j)
            geo.append((ln, dst * seg + off, src * seg + off))
        else:
            raise ValueError(kind)
    return geo


# --------------------------------------------------------------------------
# schedule helpers
# --------------------------------------------------------------------------
def _phases(sched: dict) -> List[dict]:
    return sched["phases"] if "phases" in sched else [sched]


def _c_topo(t: dict):
    offs, edges, bounds = [0], [], []
    for c in t["constraints"]:
        for e in c["edges"]:
            edges += [int(e[0]), int(e[1])]
        offs.append(len(edges) // 2)
        bounds.append(int(c["bound"]))
    keep = [np.asarray(offs, np.int32), np.asarray(edges or [0], np.int32),
            np.asarray(bounds or [0], np.int32)]
    st = _Topo(t["P"], len(t["constraints"]), keep[0].ctypes.data, keep[1].ctypes.data,
               keep[2].ctypes.data)
    return st, keep


def _c_sched(s: dict):
    rounds = np.asarray(s["rounds"] or [0], np.int32)
    sends = np.asarray(s["sends"] or [[0, 0, 0, 0]], np.int32).reshape(-1, 4)
    st = _Sched(s["G"], s["S"], rounds.ctypes.data, len(s["sends"]), sends.ctypes.data)
    return st, [rounds, sends]


def verify(sched: dict, topo: Optional[dict] = None) -> List[Tuple[str, int, int, int, int]]:
    """Verify every phase; returns violations as (kind, step, chunk, src, dst)."""
    out = []
    for ph in _phases(sched):
        tj = ph["topology"]
        t = topo or ({"name": tj["name"], "P": ph["P"], "constraints": tj["constraints"]}
                     if "constraints" in tj else topology_by_name(tj["name"]))
        P, G = ph["P"], ph["G"]
        kind = ph["collective"]
        a, b = pre_post(kind, G, P, ph.get("root", 0) or 0)
        tst, k1 = _c_topo(t)
        sst, k2 = _c_sched(ph)
        buf = (_Viol * 4096)()
        fn = lib().oracle_verify_combining if kind in COMBINING else lib().oracle_verify
        n = fn(ctypes.byref(tst), ctypes.byref(sst), a.ctypes.data_as(ctypes.c_void_p),
               b.ctypes.data_as(ctypes.c_void_p), buf, 4096)
        out += [(V_NAMES[v.kind], v.step, v.chunk, v.src, v.dst) for v in buf[:min(n, 4096)]]
    return out


def _run_phase(ph: dict, slots: List[np.ndarray], present: np.ndarray, off, ln, dtype: int,
               nthreads: int):
    P = ph["P"]
    sst, keep = _c_sched(ph)
    ptrs = (ctypes.c_void_p * P)(*[s.ctypes.data for s in slots])
    r = lib().oracle_execute(ctypes.c_int32(P), ctypes.byref(sst),
                             ctypes.c_int(1 if ph["collective"] in COMBINING else 0),
                             ctypes.c_int(dtype), off.ctypes.data_as(ctypes.c_void_p),
                             ln.ctypes.data_as(ctypes.c_void_p), ptrs,
                             present.ctypes.data_as(ctypes.c_void_p), ctypes.c_int(nthreads))
    if r != 0:
        raise ValueError("oracle_execute rejected its arguments")


class Execution:
    """One execution of a schedule (or composition) over the payload model
    of SPEC.md:393-397: per-node chunk slots packed from the per-rank input
    buffers by the Appendix C layout.  ``run`` is the timed executor loop
    (the C restatement of SPEC.md:418-426); packing/unpacking is layout
    plumbing around it."""

    def __init__(self, sched: dict, inputs: Sequence[np.ndarray], nbytes: int, dtype: int = U8,
                 check: bool = True):
        if check:
            v = verify(sched)
            if v:
                raise ValueError(f"unverified schedule rejected (SPEC.md:420): {v[:4]}")
        self.sched = sched
        self.kind = sched["collective"]
        self.phases = _phases(sched)
        self.P = P = sched["P"]
        self.root = sched.get("root", 0) or 0
        self.G = G = self.phases[-1]["G"]
        self.dtype = dtype
        self.nbytes = nbytes
        C_geo = G // P if self.kind not in ("broadcast", "reduce") else G
        self.geo = geo = chunk_geometry(self.kind, P, C_geo, nbytes, G)
        self.ln = np.asarray([g[0] for g in geo], np.int64)
        self.off = np.zeros(G, np.int64)
        if G:
            self.off[1:] = np.cumsum(self.ln)[:-1]
        total = int(self.ln.sum())
        self.slots = [np.zeros(max(total, 1), np.uint8) for _ in range(P)]
        self.inputs = inputs
        pre, _ = pre_post(self.phases[0]["collective"], self.phases[0]["G"], P, self.root)
        self.pre = pre
        self.combining_first = self.phases[0]["collective"] in COMBINING
        self.present = np.zeros((P, G), np.uint8)
        self.pack()

    def pack(self):
        for c in range(self.G):
            L, io = int(self.ln[c]), self.geo[c][1]
            o = int(self.off[c])
            for n in range(self.P):
                if self.pre[c, n]:
                    self.slots[n][o:o + L] = self.inputs[n][io:io + L]
        self.present[:] = self.pre.T

    def run(self, nthreads: int = 1):
        """The executor proper; re-packs first when the previous run reduced
        into the slots (combining phases are not idempotent)."""
        if getattr(self, "_dirty", False):
            self.pack()
        self.present[:] = self.pre.T
        for k, ph in enumerate(self.phases):
            if k > 0:  # composition: the next phase starts from its own pre
                p2, _ = pre_post(ph["collective"], ph["G"], self.P, self.root)
                self.present[:] = p2.T
            _run_phase(ph, self.slots, self.present, self.off, self.ln, self.dtype, nthreads)
        self._dirty = any(ph["collective"] in COMBINING for ph in self.phases)

    def outputs(self, outputs: Optional[Sequence[np.ndarray]] = None) -> List[np.ndarray]:
        _, rb = buffer_sizes(self.kind, self.P, self.nbytes)
        if outputs is None:
            outputs = [np.zeros(rb, np.uint8) for _ in range(self.P)]
        last = self.phases[-1]
        _, post = pre_post(last["collective"], last["G"], self.P, self.root)
        for c in range(self.G):
            L, oo, o = int(self.ln[c]), self.geo[c][2], int(self.off[c])
            for n in range(self.P):
                if post[c, n]:
                    if not self.present[n, c]:
                        raise ValueError(f"chunk {c} missing at node {n}")
                    outputs[n][oo:oo + L] = self.slots[n][o:o + L]
        return outputs


def execute(sched: dict, inputs: Sequence[np.ndarray], nbytes: int, dtype: int = U8,
            nthreads: int = 1, check: bool = True,
            outputs: Optional[Sequence[np.ndarray]] = None) -> List[np.ndarray]:
    """Run the schedule on per-rank input byte buffers; returns per-rank output
    byte buffers laid out as the GPU executor lays them out (Appendix C).
    Output bytes no chunk covers keep their initial value (zero, or the
    ``outputs`` passed in)."""
    ex = Execution(sched, inputs, nbytes, dtype, check)
    ex.run(nthreads)
    if outputs is not None:
        outputs = [np.array(o, dtype=np.uint8, copy=True) for o in outputs]
    return ex.outputs(outputs)


# --------------------------------------------------------------------------
# second restatement (pure Python, small cases only)
# --------------------------------------------------------------------------
def _reduce_py(dtype: int, acc: Optional[np.ndarray], ins: List[np.ndarray]) -> np.ndarray:
    dt = NP_DTYPE[dtype]
    vals = [x.view(dt) for x in ins]
    if dtype in (U8, I32):
        a = (acc.view(dt).copy() if acc is not None else vals[0].copy())
        for v in (vals if acc is not None else vals[1:]):
            a = (a + v).astype(dt)
        return a.view(np.uint8)
    if dtype == F32:
        a = acc.view(np.float32).copy() if acc is not None else vals[0].copy()
        with np.errstate(invalid="ignore", over="ignore"):
            for v in (vals if acc is not None else vals[1:]):
                a = (a + v).astype(np.float32)
        a = a.view(np.uint32)
        a[np.isnan(a.view(np.float32))] = 0x7FFFFFFF  # canonical NaN, as GPU arithmetic returns it
        return a.view(np.uint8)
    # bf16 / f16: widen to f32, add in order, round once
    def widen(x):
        if dtype == BF16:
            return (x.astype(np.uint32) << 16).view(np.float32)
        return x.astype(np.float32)
    a = widen(acc.view(dt)) if acc is not None else widen(vals[0])
    with np.errstate(invalid="ignore", over="ignore"):
        for v in (vals if acc is not None else vals[1:]):
            a = (a + widen(v)).astype(np.float32)
    if dtype == BF16:
        u = a.view(np.uint32).astype(np.uint64)
        r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
        r[np.isnan(a)] = 0x7FFF
        return r.view(np.uint8)
    with np.errstate(invalid="ignore", over="ignore"):
        r = a.astype(np.float16).view(np.uint16)
    r[np.isnan(a)] = 0x7FFF  # canonical NaN (PTX cvt)
    return r.view(np.uint8)


def execute_py(sched: dict, inputs: Sequence[np.ndarray], nbytes: int, dtype: int = U8):
    """Independent pure-Python restatement of execute that
    works directly on (node, chunk) -> bytes dictionaries."""
    kind = sched["collective"]
    phases = _phases(sched)
    P = sched["P"]
    root = sched.get("root", 0) or 0
    G = phases[-1]["G"]
    C_geo = G // P if kind not in ("broadcast", "reduce") else G
    geo = chunk_geometry(kind, P, C_geo, nbytes, G)
    val: Dict[Tuple[int, int], np.ndarray] = {}
    pre, _ = pre_post(phases[0]["collective"], G, P, root)
    for c in range(G):
        for n in range(P):
            if pre[c, n]:
                L, io, _ = geo[c]
                val[(c, n)] = np.array(inputs[n][io:io + L], np.uint8)
    for k, ph in enumerate(phases):
        comb = ph["collective"] in COMBINING
        have = set(val.keys())
        if k > 0:
            p2, _ = pre_post(ph["collective"], G, P, root)
            have = {(c, n) for c in range(G) for n in range(P) if p2[c, n]}
        for s in range(ph["S"]):
            sends = sorted((t for t in ph["sends"] if t[3] == s), key=lambda t: (t[2], t[0], t[1]))
            snap = {key: v.copy() for key, v in val.items()}
            new_have = set(have)
            groups: Dict[Tuple[int, int], List[int]] = {}
            for c, a, b, _ in sends:
                if (c, a) not in have:
                    continue
                if comb:
                    groups.setdefault((c, b), []).append(a)
                else:
                    val[(c, b)] = snap[(c, a)].copy()
                new_have.add((c, b))
            for (c, b), srcs in groups.items():
                old = snap[(c, b)] if (c, b) in have else None
                val[(c, b)] = _reduce_py(dtype, old, [snap[(c, a)] for a in srcs])
            have = new_have
    _, post = pre_post(phases[-1]["collective"], G, P, root)
    sb, rb = buffer_sizes(kind, P, nbytes)
    outs = [np.zeros(rb, np.uint8) for _ in range(P)]
    for c in range(G):
        for n in range(P):
            if post[c, n]:
                L, _, oo = geo[c]
                outs[n][oo:oo + L] = val[(c, n)]
    return outs


# --------------------------------------------------------------------------
# seeded inputs + digests (shared with tests and bench)
# --------------------------------------------------------------------------
def seeded_inputs(kind: str, P: int, nbytes: int, dtype: int, seed: int,
                  mode: str = "random") -> List[np.ndarray]:
    """Deterministic per-rank input buffers (bytes).  mode 'random' = uniform
    bytes (u8), uniform [-1,1) floats, or full-range ints; 'smallint' =
    integers in [-16,16] (exact under any summation order); 'bits' = uniform
    bit patterns for the float types (special values included)."""
    sb, _ = buffer_sizes(kind, P, nbytes)
    es = ESIZE[dtype]
    out = []
    for r in range(P):
        rng = np.random.default_rng([seed, r])
        n = sb // es
        if mode == "bits" and dtype in (F16, BF16, F32):
            # every bit pattern: subnormals, infinities, NaNs, the largest finite values
            arr = rng.integers(0, 2**(8 * es), size=n, dtype=np.uint64).astype({2: np.uint16, 4: np.uint32}[es])
        elif mode == "smallint":
            v = rng.integers(-16, 17, size=n)
            arr = {U8: v.astype(np.uint8), I32: v.astype(np.int32), F32: v.astype(np.float32),
                   F16: v.astype(np.float16),
                   BF16: (v.astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)}[dtype]
        elif dtype == U8:
            arr = rng.integers(0, 256, size=n, dtype=np.uint8)
        elif dtype == I32:
            arr = rng.integers(-2**31, 2**31, size=n, dtype=np.int64).astype(np.int32)
        elif dtype == F32:
            arr = rng.uniform(-1, 1, size=n).astype(np.float32)
        elif dtype == F16:
            arr = rng.uniform(-1, 1, size=n).astype(np.float16)
        else:
            f = rng.uniform(-1, 1, size=n).astype(np.float32)
            arr = (f.view(np.uint32) >> 16).astype(np.uint16)
        b = arr.view(np.uint8)
        pad = np.zeros(sb, np.uint8)
        pad[:b.size] = b
        out.append(pad)
    return out


def cli_payload(nbytes: int, seed: int, rank: int) -> np.ndarray:
    """Input bytes the C++ CLI (sccl-exec exec) generates: little-endian
    bytes of splitmix64((seed << 40) ^ (rank << 32) ^ word)."""
    M = 0xFFFFFFFFFFFFFFFF
    nw = (nbytes + 7) // 8
    x = ((np.uint64(seed) << np.uint64(40)) ^ (np.uint64(rank) << np.uint64(32))
         ^ np.arange(nw, dtype=np.uint64))
    with np.errstate(over="ignore"):
        x = x + np.uint64(0x9e3779b97f4a7c15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xbf58476d1ce4e5b9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94d049bb133111eb)
        x = x ^ (x >> np.uint64(31))
    return x.view(np.uint8)[:nbytes].copy()


def fnv1a(b: np.ndarray) -> str:
    h = 0xcbf29ce484222325
    for c in np.ascontiguousarray(b).view(np.uint8).tobytes():
        h ^= c
        h = (h * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return f"{h:016x}"


def digest(bufs: Sequence[np.ndarray]) -> str:
    h = hashlib.sha256()
    for b in bufs:
        h.update(np.ascontiguousarray(b).view(np.uint8).tobytes())
    return h.hexdigest()


def load_schedule(path: str) -> dict:
    with open(path) as f:
        return json.load(f)
