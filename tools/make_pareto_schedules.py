#!/usr/bin/env python3
"""BASELINE config 5: Pareto frontiers (Algorithm 1) of
allgather on ring(P) for k = 0..3, on full(P), and on the NVSwitch model
switch(P) (per-GPU egress / ingress groups) for k = 0 and
k = P - 2, P in {2, 4, 8}; each
frontier entry is committed as a canonical schedule file (models are not
unique) under paper_2008_08708_b200/frontiers/, with an index.
Usage: python tools/make_pareto_schedules.py"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2008_08708_b200 import synth  # noqa: E402

OUT = os.path.join(ROOT, "paper_2008_08708_b200", "frontiers")


def main():
    os.makedirs(OUT, exist_ok=True)
    index = []
    for P in (2, 4, 8):
        runs = [(f"ring:{P}", k) for k in range(4)] + [(f"full:{P}", 0)]
        runs += [(f"switch:{P}", k) for k in sorted({0, P - 2})]
        for topo, k in runs:
            fr = synth.pareto_synthesize("allgather", topo, k, max_steps=8, timeout=120)
            for e in fr:
                name = f"ag_{topo.replace(':', '')}_k{k}_{e['C']}_{e['S']}_{e['R']}"
                with open(os.path.join(OUT, name + ".json"), "w") as f:
                    f.write(e["schedule"] + "\n")
                index.append({"file": name + ".json", "P": P, "topology": topo, "k": k, "C": e["C"], "S": e["S"],
                              "R": e["R"], "R_over_C": e["ratio"], "bandwidth_optimal": e["bandwidth_optimal"],
                              "solver_seconds": e["seconds"]})
                print(index[-1], flush=True)
    with open(os.path.join(OUT, "index.json"), "w") as f:
        json.dump(index, f, indent=1)


if __name__ == "__main__":
    main()
