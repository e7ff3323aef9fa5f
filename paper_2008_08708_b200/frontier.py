"""Topology discovery -> synthesis target -> candidate schedules -> per-size
choice: SURVEY.md 8(f) rows f2, f1 and f3 wired together.

The reference "probes the target hardware topology" and synthesizes for it
(PAPER.md:175-177), then "automatically switch[es] between multiple
implementations based on the input size".  Here:

  * ``topology.discover()`` (f2) names the machine: ``switch:N`` on an
    NVSwitch box, ``full:N`` for plain all-to-all peer access,
    ``loopback:1`` on one GPU;
  * the candidates (f1) are the Pareto frontiers of Algorithm 1 for that
    target, committed under ``frontiers/`` (index.json: topology, k,
    (C,S,R)) -- schedules are not unique, so execution always
    uses the committed files -- or, for a target with no committed
    frontier, a fresh ``synth.pareto_synthesize`` run;
  * ``sccl.select`` (f3) picks the schedule and protocol per buffer size
    with the fitted B200 cost model of that kind of plan.

On an NVSwitch box every pair of GPUs is connected, so the full(N)
frontier's schedules are valid there too (they describe the same sends
under per-pair rather than per-GPU bandwidth accounting); both are
candidates.  In loopback the ranks share one HBM and no link model
applies: every committed frontier for the rank count is a candidate.
"""
from __future__ import annotations

import json
import os
from typing import Dict, List, Optional, Sequence, Tuple

from . import sccl
from . import topology as _topology

FRONTIER_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "frontiers")


def index() -> List[dict]:
    with open(os.path.join(FRONTIER_DIR, "index.json")) as f:
        return json.load(f)


def committed(topo: str, collective: str = "allgather") -> List[Tuple[dict, str]]:
    """(index entry, canonical schedule JSON) of every committed frontier
    entry for a topology (all k), deduplicated by (C, S, R)."""
    if collective != "allgather":
        raise ValueError("frontiers are allgather schedules; allreduce candidates are derived from them")
    out, seen = [], set()
    for e in index():
        if e["topology"] != topo:
            continue
        key = (e["C"], e["S"], e["R"])
        if key in seen:
            continue
        seen.add(key)
        with open(os.path.join(FRONTIER_DIR, e["file"])) as f:
            out.append((e, f.read().strip()))
    return out


def targets_for(target: str, P: Optional[int] = None) -> List[str]:
    """Topologies whose frontiers are candidates on a discovered target."""
    kind, _, n = target.partition(":")
    if kind == "loopback":
        if not P:
            raise ValueError("loopback needs the rank count P")
        return [f"switch:{P}", f"full:{P}", f"ring:{P}"]
    if kind == "switch":
        return [target, f"full:{n}"]
    if kind in ("full", "ring"):
        return [target]
    raise ValueError(f"no synthesis target for {target!r}")


def candidates(collective: str, target: str, P: Optional[int] = None, synthesize_missing: bool = False,
               k: int = 0) -> List[str]:
    """Candidate schedules (canonical JSON) of `collective` for a discovered
    target.  allreduce candidates are the RS+AG compositions of the
    allgather frontier entries."""
    ags: List[str] = []
    for topo in targets_for(target, P):
        entries = committed(topo)
        if not entries and synthesize_missing:
            from . import synth
            entries = [({"C": e["C"], "S": e["S"], "R": e["R"]}, e["schedule"])
                       for e in synth.pareto_synthesize("allgather", topo, k)]
        ags += [js for _, js in entries]
    if not ags:
        raise ValueError(f"no committed frontier for {target} (P={P}); pass synthesize_missing=True")
    ags = list(dict.fromkeys(ags))
    if collective == "allgather":
        return ags
    if collective == "allreduce":
        return [sccl.compose_allreduce(sccl.invert(js), js) for js in ags]
    raise ValueError(f"unsupported collective {collective!r}")


def for_this_machine(collective: str = "allgather", P: Optional[int] = None,
                     ndev: Optional[int] = None) -> Tuple[Dict, List[str]]:
    """(discovery record, candidate schedules) for the GPUs this process sees.
    One GPU is a loopback target with P ranks (default 8)."""
    info = _topology.discover(ndev)
    target = info["target"]
    if target == "unknown":
        raise RuntimeError(f"topology discovery found no usable target: {info}")
    if target.startswith("loopback"):
        P = P or 8
    else:
        P = P or int(target.split(":")[1])
    info["candidate_topologies"] = targets_for(target, P)
    return info, candidates(collective, target, P)


def choose(schedules: Sequence[str], bytes_per_rank: int, dtype: int = sccl.U8,
           multiprocess: bool = False) -> Tuple[int, str, float]:
    """The cost model's choice for one size: (index, protocol, predicted us)."""
    return sccl.select(list(schedules), bytes_per_rank, dtype, multiprocess)
