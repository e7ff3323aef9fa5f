"""SMT synthesis of k-synchronous schedules (host prerequisite).

Restates the reference's encoding module
and solver driver: the instance (G,S,R,P,B,pre,post) becomes
a QF_LIA problem with
  start_c_n in [0,S+1]      earliest step chunk c is at node n (S+1 = never)
  snd_n_c_m  (n,m) in E     node n sends c to m at some step
  r_s >= 1                  rounds of step s
and constraints C1-C6; an SMT-LIB2 solver (Z3, SCCL_SOLVER) runs as a child
process over stdin; the model decodes to T = {(c,n,m,t) | snd_n_c_m and
start_c_m = t+1} and Q = (r_1..r_S), which is verified by the C++ verifier
before it is returned.  Variable names follow SPEC.md:254-255
(st_c_n, snd_n_c_n', r_s).

Used to produce the schedules the benchmark configurations name that have
no hand construction: (C,S,R) = (2,4,7) on ring(8) (Table 5)
and the DGX-1 (6,3,7) allgather whose composition is the (48,6,14)
allreduce of SPEC.md:426 / acceptance :641.
"""
from __future__ import annotations

import os
import re
import subprocess
import time
from typing import Dict, List, Optional, Tuple

from . import sccl

def topology_edges(name: str) -> Tuple[int, List[Tuple[List[Tuple[int, int]], int]]]:
    """(P, [(edges, bound)]) of a named topology: the builders of
    SPEC.md:36-71 restated (the C++ library rebuilds the same constraints
    when it verifies the decoded schedule, so a disagreement fails loudly)."""
    P = {"dgx1": 8, "amd-z52": 8}.get(name) or int(name.split(":")[1])
    # builders restated; E and groups per PAPER.md:343-345
    if name in ("dgx1",):
        bw = {}
        for cyc, b in (((0, 1, 4, 5, 6, 7, 2, 3), 2), ((0, 2, 1, 3, 6, 4, 7, 5), 1)):
            for i in range(8):
                a, d = cyc[i], cyc[(i + 1) % 8]
                bw[(a, d)] = bw.get((a, d), 0) + b
                bw[(d, a)] = bw.get((d, a), 0) + b
        return P, [([e], b) for e, b in sorted(bw.items())]
    kind = "ring" if name == "amd-z52" else name.split(":")[0]
    if kind == "ring":
        es = sorted({(i, (i + 1) % P) for i in range(P)} | {((i + 1) % P, i) for i in range(P)})
        return P, [([e], 1) for e in es]
    if kind == "full":
        return P, [([(a, b)], 1) for a in range(P) for b in range(P) if a != b]
    if kind == "switch":
        g = [([(n, d) for d in range(P) if d != n], 1) for n in range(P)]
        g += [([(s, n) for s in range(P) if s != n], 1) for n in range(P)]
        return P, g
    raise ValueError(name)


def _relations(kind: str, G: int, P: int, root: int):
    rel = {"all": lambda c: set(range(P)), "root": lambda c: {root},
           "scattered": lambda c: {c % P}, "transpose": lambda c: {(c // P) % P}}
    pre, post = {"allgather": ("scattered", "all"), "gather": ("scattered", "root"),
                 "alltoall": ("scattered", "transpose"), "broadcast": ("root", "all"),
                 "scatter": ("root", "scattered")}[kind]
    return ({(c, n) for c in range(G) for n in rel[pre](c)}, {(c, n) for c in range(G) for n in rel[post](c)})


def encode(kind: str, topo: str, C: int, S: int, R: int, root: int = 0) -> Tuple[str, dict]:
    """SMT-LIB2 text of C1-C6."""
    P, groups = topology_edges(topo)
    G = C if kind == "broadcast" else P * C
    pre, post = _relations(kind, G, P, root)
    E = sorted({e for es, b in groups for e in es
                if all(bb > 0 for ees, bb in groups if e in ees)})
    L = ["(set-logic QF_LIA)"]
    st = lambda c, n: f"st_{c}_{n}"
    snd = lambda n, c, m: f"snd_{n}_{c}_{m}"
    for c in range(G):
        for n in range(P):
            L.append(f"(declare-fun {st(c, n)} () Int)")
            L.append(f"(assert (and (>= {st(c, n)} 0) (<= {st(c, n)} {S + 1})))")
    for (n, m) in E:
        for c in range(G):
            L.append(f"(declare-fun {snd(n, c, m)} () Bool)")
    for s in range(1, S + 1):
        L.append(f"(declare-fun r_{s} () Int)")
        L.append(f"(assert (>= r_{s} 1))")
    # C1, C2
    for (c, n) in pre:
        L.append(f"(assert (= {st(c, n)} 0))")
    for (c, n) in post:
        L.append(f"(assert (<= {st(c, n)} {S}))")
    # C3 (with the converse)
    for c in range(G):
        for n in range(P):
            if (c, n) in pre:
                continue
            ins = [snd(a, c, n) for (a, b) in E if b == n]
            tot = "(+ " + " ".join(f"(ite {x} 1 0)" for x in ins) + " 0)" if ins else "0"
            L.append(f"(assert (=> (<= {st(c, n)} {S}) (= {tot} 1)))")
            L.append(f"(assert (=> (= {st(c, n)} {S + 1}) (= {tot} 0)))")
    # C4
    for (n, m) in E:
        for c in range(G):
            L.append(f"(assert (=> {snd(n, c, m)} (< {st(c, n)} {st(c, m)})))")
    # C5
    for s in range(1, S + 1):
        for es, b in groups:
            terms = [f"(ite (and {snd(n, c, m)} (= {st(c, m)} {s})) 1 0)" for (n, m) in es if (n, m) in E
                     for c in range(G)]
            if terms:
                L.append(f"(assert (<= (+ {' '.join(terms)}) (* {b} r_{s})))")
    # C6
    L.append(f"(assert (= (+ {' '.join(f'r_{s}' for s in range(1, S + 1))}) {R}))")
    L.append("(check-sat)")
    L.append("(get-model)")
    meta = {"kind": kind, "topo": topo, "P": P, "G": G, "C": C, "S": S, "R": R, "root": root, "E": E}
    return "\n".join(L) + "\n", meta


def solve(text: str, timeout: float = 600.0) -> Tuple[str, Dict[str, str], float]:
    """Run the SMT-LIB2 solver child process."""
    solver = os.environ.get("SCCL_SOLVER", "z3")
    args = os.environ.get("SCCL_SOLVER_ARGS", "-in -smt2").split()
    t0 = time.time()
    try:
        out = subprocess.run([solver] + args, input=text, capture_output=True, text=True, timeout=timeout).stdout
    except subprocess.TimeoutExpired:
        return "unknown", {}, time.time() - t0
    dt = time.time() - t0
    status = out.strip().split("\n", 1)[0].strip()
    model = {}
    for m in re.finditer(r"\(define-fun\s+(\S+)\s+\(\)\s+\w+\s+(\S+?)\)", out):
        model[m.group(1)] = m.group(2)
    return status, model, dt


def decode(model: Dict[str, str], meta: dict) -> dict:
    """Q, T from the model (start = t+1)."""
    S, G = meta["S"], meta["G"]
    sends = []
    for (n, m) in meta["E"]:
        for c in range(G):
            if model.get(f"snd_{n}_{c}_{m}") == "true":
                t = int(model[f"st_{c}_{m}"]) - 1
                if 0 <= t < S:
                    sends.append([c, n, m, t])
    rounds = [int(model[f"r_{s}"]) for s in range(1, S + 1)]
    d = {"collective": meta["kind"], "version": 1, "topology": {"name": meta["topo"]}, "P": meta["P"],
         "G": G, "C": meta["C"], "S": S, "R": meta["R"]}
    if meta["kind"] in ("broadcast", "gather", "scatter"):
        d["root"] = meta["root"]
    d["rounds"] = rounds
    d["sends"] = sorted(sends, key=lambda x: (x[3], x[0], x[1], x[2]))
    return d


def synthesize(kind: str, topo: str, C: int, S: int, R: int, root: int = 0,
               timeout: float = 600.0) -> Tuple[str, Optional[str], float]:
    """Returns (status, canonical schedule JSON or None, solver seconds)."""
    text, meta = encode(kind, topo, C, S, R, root)
    status, model, dt = solve(text, timeout)
    if status != "sat":
        return status, None, dt
    js = sccl.canonicalize(decode(model, meta))
    v = sccl.verify(js)
    if v:
        raise RuntimeError(f"decoded schedule failed verification: {v[:3]}")
    return "sat", js, dt


# ----------------------------------------------------------------------------
# Algorithm 1, Pareto-Synthesize
# ----------------------------------------------------------------------------
def diameter(topo: str) -> int:
    """Max over node pairs of the shortest directed path over E."""
    P, groups = topology_edges(topo)
    E = {e for es, b in groups for e in es if b > 0}
    best = 0
    for s in range(P):
        dist = {s: 0}
        frontier = [s]
        while frontier:
            nxt = []
            for u in frontier:
                for (a, b) in E:
                    if a == u and b not in dist:
                        dist[b] = dist[u] + 1
                        nxt.append(b)
            frontier = nxt
        if len(dist) < P:
            raise ValueError(f"unreachable pair from node {s} in {topo}")
        best = max(best, max(dist.values()))
    return best


def bandwidth_lower_bound(kind: str, topo: str, root: int = 0) -> "Fraction":
    """Per-node bound on R/C (the paper's section 2.4
    argument): a node that must receive X chunks (per per-node chunk) over
    ingress bandwidth B, or send X over egress bandwidth B, needs
    R/C >= X / B.  Gather concentrates the (P-1) receipts on the root's
    ingress, scatter and broadcast the root's sends on its egress.  (The
    exhaustive cut bounds of SPEC.md:100 are not restated; the per-node bound
    is sound.)  Always > 0 for P > 1."""
    from fractions import Fraction
    P, groups = topology_edges(topo)
    others = [n for n in range(P) if n != root]
    need_in = {n: Fraction(0) for n in range(P)}
    need_out = {n: Fraction(0) for n in range(P)}
    if kind == "allgather":
        need_in = {n: Fraction(P - 1) for n in range(P)}
    elif kind == "alltoall":
        need_in = {n: Fraction(P - 1, P) for n in range(P)}
    elif kind == "broadcast":
        need_in.update({n: Fraction(1) for n in others})
        need_out[root] = Fraction(1)
    elif kind == "gather":
        need_in[root] = Fraction(P - 1)
    elif kind == "scatter":
        need_out[root] = Fraction(P - 1)
    else:
        raise ValueError(f"no bandwidth bound for {kind}")

    def cap(n, inbound):
        side = (lambda e: e[1] == n) if inbound else (lambda e: e[0] == n)
        c = sum(b for es, b in groups for e in es if side(e) and len(es) == 1)
        for es, b in groups:  # grouped ingress / egress constraints (switch model)
            if len(es) > 1 and all(side(e) for e in es):
                c = b if c == 0 else min(c, b)
        return c

    best = Fraction(0)
    for n in range(P):
        for need, inbound in ((need_in[n], True), (need_out[n], False)):
            c = cap(n, inbound)
            if need and c:
                best = max(best, need / c)
    if best <= 0:
        raise ValueError(f"{kind} on {topo}: no positive bandwidth bound (P = {P})")
    return best


def pareto_synthesize(kind: str, topo: str, k: int, max_steps: int = 8, timeout: float = 120.0,
                      root: int = 0) -> List[dict]:
    """Algorithm 1: for S = diameter.. try (R, C) with S <= R <= S+k and
    R/C >= b_l in ascending R/C (ties: smaller R); report the first SAT per
    S; stop once R/C reaches b_l."""
    from fractions import Fraction
    a_l = diameter(topo)
    b_l = bandwidth_lower_bound(kind, topo, root)  # > 0, so every (R, C) scan below ends
    frontier: List[dict] = []
    best_ratio = None
    for S in range(a_l, max_steps + 1):
        cands = []
        for R in range(S, S + k + 1):
            C = 1
            while Fraction(R, C) >= b_l:
                if best_ratio is None or Fraction(R, C) < best_ratio:
                    cands.append((Fraction(R, C), R, C))
                C += 1
        cands.sort()
        for ratio, R, C in cands:
            if kind == "alltoall" and C % topology_edges(topo)[0]:
                continue
            st, js, dt = synthesize(kind, topo, C, S, R, root, timeout)
            if st == "sat":
                frontier.append({"C": C, "S": S, "R": R, "ratio": str(ratio), "seconds": round(dt, 2),
                                 "schedule": js, "bandwidth_optimal": ratio == b_l})
                best_ratio = ratio
                break
        if best_ratio is not None and best_ratio == b_l:
            break
    return frontier
