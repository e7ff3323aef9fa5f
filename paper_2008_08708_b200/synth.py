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


def automorphisms(topo: str) -> List[Tuple[int, ...]]:
    """Node permutations that preserve every constraint of the topology
    (edge sets with their bounds)."""
    import itertools
    P, groups = topology_edges(topo)
    cons = {(frozenset(es), b) for es, b in groups}
    out = []
    for g in itertools.permutations(range(P)):
        if all((frozenset((g[a], g[d]) for a, d in es), b) in cons for es, b in cons):
            out.append(g)
    return out


def encode_symmetric(kind: str, topo: str, C: int, S: int, R: int, group: List[Tuple[int, ...]],
                     root: int = 0) -> Tuple[str, dict]:
    """C1-C6 restricted to schedules invariant under a node-permutation
    group acting freely on the nodes (an automorphism group of the
    topology): chunk (i, n) -- index i of node n -- is sent along the image
    under g of the route of chunk (i, g^-1(n)).  Variables exist only for
    the chunks of one node per orbit; the bandwidth constraint C5 counts the
    images of every base send.  A |G|-fold smaller problem; a solution is a
    valid schedule (decode_symmetric expands and the C++ verifier checks
    it), but symmetry may exclude every solution (then: unsat here, not
    necessarily for the instance)."""
    if kind not in ("allgather", "alltoall"):
        raise ValueError("symmetric encoding: per-node chunk ownership (allgather, alltoall) only")
    P, groups = topology_edges(topo)
    if any(g[n] == n for g in group[1:] for n in range(P)) or group[0] != tuple(range(P)):
        raise ValueError("the group must start with the identity and act freely on the nodes")
    G = P * C
    pre, post = _relations(kind, G, P, root)
    E = sorted({e for es, b in groups for e in es if all(bb > 0 for ees, bb in groups if e in ees)})
    reps, seen = [], set()
    for n in range(P):
        if n not in seen:
            reps.append(n)
            seen |= {g[n] for g in group}
    inv = [tuple(sorted(range(P), key=lambda x: g[x])) for g in group]  # g^-1
    base = [i * P + n for n in reps for i in range(C)]
    L = ["(set-logic QF_LIA)"]
    st = lambda c, n: f"st_{c}_{n}"
    snd = lambda n, c, m: f"snd_{n}_{c}_{m}"
    for c in base:
        for n in range(P):
            L.append(f"(declare-fun {st(c, n)} () Int)")
            L.append(f"(assert (and (>= {st(c, n)} 0) (<= {st(c, n)} {S + 1})))")
        for (n, m) in E:
            L.append(f"(declare-fun {snd(n, c, m)} () Bool)")
    for s_ in range(1, S + 1):
        L.append(f"(declare-fun r_{s_} () Int)")
        L.append(f"(assert (>= r_{s_} 1))")
    for c in base:
        for n in range(P):
            if (c, n) in pre:
                L.append(f"(assert (= {st(c, n)} 0))")
            if (c, n) in post:
                L.append(f"(assert (<= {st(c, n)} {S}))")
            if (c, n) not in pre:
                ins = [snd(a, c, n) for (a, b) in E if b == n]
                tot = "(+ " + " ".join(f"(ite {x} 1 0)" for x in ins) + " 0)" if ins else "0"
                L.append(f"(assert (=> (<= {st(c, n)} {S}) (= {tot} 1)))")
                L.append(f"(assert (=> (= {st(c, n)} {S + 1}) (= {tot} 0)))")
        for (n, m) in E:
            L.append(f"(assert (=> {snd(n, c, m)} (< {st(c, n)} {st(c, m)})))")
    for s_ in range(1, S + 1):
        for es, b in groups:
            terms = []
            for gi in inv:  # send (n,m) of image chunk g(c) <=> send (g^-1 n, g^-1 m) of base chunk c
                for (n, m) in es:
                    a_, d_ = gi[n], gi[m]
                    if (a_, d_) in E:
                        terms += [f"(ite (and {snd(a_, c, d_)} (= {st(c, d_)} {s_})) 1 0)" for c in base]
            if terms:
                L.append(f"(assert (<= (+ {' '.join(terms)}) (* {b} r_{s_})))")
    L.append(f"(assert (= (+ {' '.join(f'r_{s_}' for s_ in range(1, S + 1))}) {R}))")
    L.append("(check-sat)")
    L.append("(get-model)")
    meta = {"kind": kind, "topo": topo, "P": P, "G": G, "C": C, "S": S, "R": R, "root": root, "E": E,
            "base": base, "group": group}
    return "\n".join(L) + "\n", meta


def decode_symmetric(model: Dict[str, str], meta: dict) -> dict:
    """Expand the base chunks' sends by the group (chunk (i, n) -> (i, g(n)))."""
    P, S = meta["P"], meta["S"]
    sends = set()
    for c in meta["base"]:
        i, n0 = divmod(c, P)
        for (a, b) in meta["E"]:
            if model.get(f"snd_{a}_{c}_{b}") == "true":
                t = int(model[f"st_{c}_{b}"]) - 1
                if 0 <= t < S:
                    for g in meta["group"]:
                        sends.add((i * P + g[n0], g[a], g[b], t))
    d = {"collective": meta["kind"], "version": 1, "topology": {"name": meta["topo"]}, "P": P, "G": meta["G"],
         "C": meta["C"], "S": S, "R": meta["R"], "rounds": [int(model[f"r_{s_}"]) for s_ in range(1, S + 1)]}
    d["sends"] = sorted([list(x) for x in sends], key=lambda x: (x[3], x[0], x[1], x[2]))
    return d


def synthesize_symmetric(kind: str, topo: str, C: int, S: int, R: int,
                         timeout: float = 600.0) -> Tuple[str, Optional[str], float]:
    """synthesize() under the topology's automorphism group (free part):
    for the DGX-1 (order 4, two node orbits) a 4x smaller problem -- the
    (6,3,7) allgather of Table 4, whose plain encoding the solver did not
    finish in 1400 s here."""
    group = [g for g in automorphisms(topo) if g == tuple(range(len(g))) or all(g[n] != n for n in range(len(g)))]
    text, meta = encode_symmetric(kind, topo, C, S, R, group)
    status, model, dt = solve(text, timeout)
    if status != "sat":
        return status, None, dt
    js = sccl.canonicalize(decode_symmetric(model, meta))
    v = sccl.verify(js)
    if v:
        raise RuntimeError(f"decoded symmetric schedule failed verification: {v[:3]}")
    return "sat", js, dt


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
        """chunks per round node n can receive (send): every link into (out
        of) n carries at most the smallest bound of the constraints that
        contain it, and a constraint made only of n's links caps their sum"""
        side = (lambda e: e[1] == n) if inbound else (lambda e: e[0] == n)
        links = {e for es, _ in groups for e in es if side(e)}
        c = sum(min(b for es, b in groups if e in es) for e in links)
        for es, b in groups:
            if len(es) > 1 and all(side(e) for e in es):
                c = min(c, b)
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
