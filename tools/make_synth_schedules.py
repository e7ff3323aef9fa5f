#!/usr/bin/env python3
"""Synthesize the Table 4/5 schedules the configs name (SMT, Z3) and commit
them as canonical schedule files under tests/golden/schedules/.  Models are
not unique, so parity is always checked on these exact files,
never by re-synthesizing.

Usage: python tools/make_synth_schedules.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2008_08708_b200 import sccl, synth  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "schedules")
ROWS = [
    # (name, kind, topology, C, S, R, source)
    ("ag_ring8_2_4_7", "allgather", "ring:8", 2, 4, 7, "Table 5 (2,4,7) (PAPER.md:954); BASELINE config 1"),
    ("ag_amdz52_2_4_7", "allgather", "amd-z52", 2, 4, 7, "Table 5 (2,4,7), AMD Z52 ring"),
    ("ag_dgx1_2_2_3", "allgather", "dgx1", 2, 2, 3, "Table 4 (2,2,3); its AR is (16,4,6)"),
    ("ag_dgx1_1_2_2", "allgather", "dgx1", 1, 2, 2, "Table 4 (1,2,2); its AR is (8,4,4)"),
    ("a2a_dgx1_8_2_3", "alltoall", "dgx1", 8, 2, 3, "Table 4 Alltoall (8,2,3): multi-hop relays"),
    # the plain encoding did not finish in 1400 s; under the DGX-1's free
    # automorphism group (order 4) it is SAT in ~40 s
    ("ag_dgx1_6_3_7", "allgather", "dgx1", 6, 3, 7,
     "Table 4 (6,3,7), bandwidth-optimal; its AR is the (48,6,14) of SPEC.md:426 / acceptance :641", "symmetric"),
]


def main():
    """usage: make_synth_schedules.py [name ...] (default: every row)"""
    os.makedirs(OUT, exist_ok=True)
    only = set(sys.argv[1:])
    for name, kind, topo, C, S, R, src, *how in ROWS:
        if only and name not in only:
            continue
        if how == ["symmetric"]:
            st, js, dt = synth.synthesize_symmetric(kind, topo, C, S, R, timeout=1200)
        else:
            st, js, dt = synth.synthesize(kind, topo, C, S, R, timeout=600)
        assert st == "sat", (name, st)
        with open(os.path.join(OUT, name + ".json"), "w") as f:
            f.write(js + "\n")
        print(f"{name}: sat in {dt:.2f} s ({src})")
        if kind == "allgather":
            ar = sccl.compose_allreduce(sccl.invert(js), js)
            with open(os.path.join(OUT, name.replace("ag_", "ar_from_") + ".json"), "w") as f:
                f.write(ar + "\n")


if __name__ == "__main__":
    main()
