"""Hand-derived synthesized schedules and constructive
generators for the NVSwitch target.

The reference's synthesizer (SMT encoding + Z3) produces
schedules in the canonical JSON form; the executor consumes
that file and nothing else.  These generators build the same objects for the
known-answer cases and for the benchmark configurations:

  B1 recursive doubling on ring(4)
  B2 ring(4) S=2 R=2 witness
  B3 DGX-1 allgather (1,2,2)                 PAPER.md:270, Table 4 :904
  B4 one-shot allgather (1,1,1) on full(P)
  B5 direct alltoall (P,1,1) on full(P)
  B7 unidirectional ring allgather (1,P-1,P-1)
  B8 bidirectional ring allgather, (1,4,4) at P=8 (Table 5)
  hamiltonian_allgather: (P-1,P-1,P-1) on full(P) -- BASELINE config 2
      "C=S=R=7": P-1 arc-disjoint directed Hamiltonian cycles of K_P*
      (Tillson's theorem), chunk i of every rank
      travels cycle i.

Every function returns a plain dict; ``to_json`` canonicalizes it through
the C++ serializer so the bytes are exactly what the executor re-emits.
"""
from __future__ import annotations

import random
from typing import Dict, List, Optional, Sequence, Tuple

Send = Tuple[int, int, int, int]  # (chunk, src, dst, step)


def _sched(kind: str, topo: str, P: int, G: int, C: int, rounds: Sequence[int],
           sends: List[Send], root: Optional[int] = None) -> dict:
    d = {"collective": kind, "version": 1, "topology": {"name": topo}, "P": P, "G": G, "C": C,
         "S": len(rounds), "R": int(sum(rounds))}
    if root is not None:
        d["root"] = root
    d["rounds"] = list(rounds)
    d["sends"] = [list(s) for s in sorted(sends, key=lambda t: (t[3], t[0], t[1], t[2]))]
    return d


def to_json(d: dict) -> str:
    from . import sccl
    return sccl.canonicalize(d)


# ---------------------------------------------------------------- allgather
def one_shot_allgather(P: int) -> dict:
    """B4: every rank sends its chunk to every other rank at step 0."""
    sends = [(n, n, d, 0) for n in range(P) for d in range(P) if d != n]
    return _sched("allgather", f"full:{P}", P, P, 1, [1], sends)


def ring_allgather(P: int) -> dict:
    """B7: {(n, n+k, n+k+1, k) | k = 0..P-2} on ring(P)."""
    sends = [(n, (n + k) % P, (n + k + 1) % P, k) for n in range(P) for k in range(P - 1)]
    return _sched("allgather", f"ring:{P}", P, P, 1, [1] * (P - 1), sends)


def bidir_ring_allgather(P: int) -> dict:
    """B8: chunks travel both ways round the ring; S = ceil((P-1)/2)."""
    fwd, bwd = (P - 1 + 1) // 2, (P - 1) // 2
    sends = [(n, (n + k) % P, (n + k + 1) % P, k) for n in range(P) for k in range(fwd)]
    sends += [(n, (n - k) % P, (n - k - 1) % P, k) for n in range(P) for k in range(bwd)]
    return _sched("allgather", f"ring:{P}", P, P, 1, [1] * fwd, sends)


def recursive_doubling_ring4() -> dict:
    """B1 (Fig. 2): ring(4), C=1, Q=(1,2), |T|=12."""
    sends = [(0, 0, 1, 0), (1, 1, 0, 0), (2, 2, 3, 0), (3, 3, 2, 0),
             (0, 0, 3, 1), (1, 0, 3, 1), (2, 3, 0, 1), (3, 3, 0, 1),
             (0, 1, 2, 1), (1, 1, 2, 1), (2, 2, 1, 1), (3, 2, 1, 1)]
    return _sched("allgather", "ring:4", 4, 4, 1, [1, 2], sends)


def ring4_s2r2() -> dict:
    """B2: SPEC.md:530 witness for ring(4) Allgather S=2, R=2."""
    sends = [(n, n, (n + 1) % 4, 0) for n in range(4)] + [(n, n, (n - 1) % 4, 0) for n in range(4)]
    sends += [(2, 1, 0, 1), (3, 2, 1, 1), (0, 3, 2, 1), (1, 0, 3, 1)]
    return _sched("allgather", "ring:4", 4, 4, 1, [1, 1], sends)


DGX1_INTER = (5, 4, 7, 6, 1, 0, 3, 2)


def dgx1_allgather_122() -> dict:
    """B3: DGX-1 (C,S,R) = (1,2,2): step 0 n sends c=n to its quad peers and
    inter(n); step 1 n forwards c=inter(n) to its quad peers."""
    sends = []
    for n in range(8):
        quad = [q for q in range(4 * (n // 4), 4 * (n // 4) + 4) if q != n]
        sends += [(n, n, q, 0) for q in quad] + [(n, n, DGX1_INTER[n], 0)]
        sends += [(DGX1_INTER[n], n, q, 1) for q in quad]
    return _sched("allgather", "dgx1", 8, 8, 1, [1, 1], sends)


def hamiltonian_cycles(P: int, seed: int = 0) -> List[List[int]]:
    """P-1 arc-disjoint directed Hamiltonian cycles covering every arc of the
    complete symmetric digraph K_P* (exists for P != 4, 6; Tillson 1980)."""
    if P in (4, 6):
        raise ValueError("K_4* and K_6* have no Hamiltonian decomposition")
    if P == 2:
        return [[0, 1]]
    rng = random.Random(seed)
    for _attempt in range(10000):
        used = [[False] * P for _ in range(P)]
        cycles: List[List[int]] = []

        def extend(path: List[int]) -> bool:
            if len(path) == P:
                if not used[path[-1]][path[0]]:
                    return True
                return False
            nxt = [v for v in range(P) if v not in path and not used[path[-1]][v]]
            rng.shuffle(nxt)
            for v in nxt[:3]:
                used[path[-1]][v] = True
                path.append(v)
                if extend(path):
                    return True
                path.pop()
                used[path[-1]][v] = False
            return False

        ok = True
        for _ in range(P - 1):
            path = [0]
            if not extend(path):
                ok = False
                break
            used[path[-1]][path[0]] = True
            cycles.append(path)
        if ok:
            return cycles
    raise RuntimeError("no decomposition found")


def hamiltonian_allgather(P: int, seed: int = 0) -> dict:
    """(P-1, P-1, P-1) allgather on full(P): chunk i*P+n starts at rank n and
    walks Hamiltonian cycle i; every arc carries exactly one chunk per step,
    so R/C = 1 = the bandwidth lower bound of full(P,1)."""
    cyc = hamiltonian_cycles(P, seed)
    C = P - 1
    sends = []
    for i, cy in enumerate(cyc):
        pos = {v: k for k, v in enumerate(cy)}
        for n in range(P):
            c = i * P + n
            for k in range(P - 1):
                a = cy[(pos[n] + k) % P]
                b = cy[(pos[n] + k + 1) % P]
                sends.append((c, a, b, k))
    return _sched("allgather", f"full:{P}", P, P * C, C, [1] * (P - 1), sends)


# ---------------------------------------------------------------- others
def direct_alltoall(P: int, C: Optional[int] = None) -> dict:
    """B5: (P,1,1): G = P^2 (C = P): chunk c goes c%P -> (c/P)%P at step 0.
    With C = k*P, every pair exchanges k chunks (R = k)."""
    C = C or P
    G = P * C
    sends = [(c, c % P, (c // P) % P, 0) for c in range(G) if c % P != (c // P) % P]
    return _sched("alltoall", f"full:{P}", P, G, C, [C // P], sends)


def one_shot_broadcast(P: int, C: int = 1, root: int = 0) -> dict:
    sends = [(c, root, d, 0) for c in range(C) for d in range(P) if d != root]
    return _sched("broadcast", f"full:{P}", P, C, C, [C], sends, root=root)


def pipelined_chain_broadcast(P: int, C: int, root: int = 0) -> dict:
    """Chunks follow the chain root -> root+1 -> ... ; chunk c leaves the
    root at step c, so S = C + P - 2 and every link carries 1 chunk/step."""
    order = [(root + k) % P for k in range(P)]
    sends = [(c, order[k], order[k + 1], c + k) for c in range(C) for k in range(P - 1)]
    return _sched("broadcast", f"ring:{P}" if P > 2 else "full:2", P, C, C, [1] * (C + P - 2), sends,
                  root=root)


def direct_gather(P: int, root: int = 0) -> dict:
    sends = [(n, n, root, 0) for n in range(P) if n != root]
    return _sched("gather", f"full:{P}", P, P, 1, [1], sends, root=root)


def direct_scatter(P: int, root: int = 0) -> dict:
    sends = [(n, root, n, 0) for n in range(P) if n != root]
    return _sched("scatter", f"full:{P}", P, P, 1, [1], sends, root=root)


def two_node_send() -> dict:
    """2-node send (broadcast from root 0)."""
    return _sched("broadcast", "full:2", 2, 1, 1, [1], [(0, 0, 1, 0)], root=0)


# ---------------------------------------------------------------- combining
def reducescatter_from(ag: dict) -> str:
    from . import sccl
    return sccl.invert(ag)


def allreduce_from(ag: dict) -> str:
    """(RS, AG) with RS = invert(AG): tuple (P*C, 2S, 2R)."""
    from . import sccl
    return sccl.compose_allreduce(sccl.invert(ag), ag)


def reduce_from(bcast: dict) -> str:
    from . import sccl
    return sccl.invert(bcast)


REGISTRY = {
    "b1": recursive_doubling_ring4,
    "b2": ring4_s2r2,
    "b3": dgx1_allgather_122,
}


def random_allgather(P: int, C: int, S: int, seed: int = 0) -> dict:
    """A random valid allgather for fuzzing the lowering and kernels: chunk
    i*P+n spreads from rank n along a random tree; a rank that gets the
    chunk at step t forwards it at some later step (so multi-hop relays,
    fan-out and uneven per-step traffic all occur).  The topology is given
    inline as the complete digraph with a bound that admits every step."""
    rng = random.Random(seed)
    G = P * C
    sends = []
    for c in range(G):
        have = {c % P: -1}  # rank -> step it received the chunk (-1: owner)
        todo = [r for r in range(P) if r != c % P]
        rng.shuffle(todo)
        for dst in todo:
            srcs = [r for r, t in have.items() if t < S - 1]
            src = rng.choice(srcs)
            step = rng.randint(have[src] + 1, S - 1)
            have[dst] = step
            sends.append((c, src, dst, step))
    bound = G
    cons = [{"edges": [[a, b]], "bound": bound} for a in range(P) for b in range(P) if a != b]
    d = _sched("allgather", f"full:{P}", P, G, C, [1] * S, sends)
    d["topology"] = {"name": f"dense:{P}", "constraints": cons}
    return d
