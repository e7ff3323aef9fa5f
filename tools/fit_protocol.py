#!/usr/bin/env python3
"""Refit the protocol model c + a*S + b*MB (plan.cpp predict_us) per
protocol from a crossover sweep (tools/tune.py lines with "protocol": ll /
simple forced), by relative-error least squares, and report the regret of
the fitted choice against the best protocol per (schedule, size).

usage: python tools/fit_protocol.py sweep.jsonl [...] [--eval llc,lla,llb,sc,sa,sb]
(--eval: also report the regret of the given constants, e.g. the policy
table's current ones)"""
import collections
import json
import sys

import numpy as np

STEPS = {"ag777": 7, "ag111": 1, "ring": 7, "ar822": 2, "ar56": 14, "ar_ring": 14, "a2a": 1}


def load(paths):
    pts = collections.defaultdict(dict)  # (sched, bytes) -> proto -> (us, MB)
    for p in paths:
        for line in open(p):
            if not line.startswith("{"):
                continue
            r = json.loads(line)
            if "us" not in r or r["sched"] not in STEPS:
                continue
            proto = r["knobs"].get("protocol", r["proto"])
            mb = r["hbm_TBps"] * r["us"]  # TB/s * us = MB of program traffic
            old = pts[(r["sched"], r["bytes"])].get(proto)
            if old is None or r["us"] < old[0]:
                pts[(r["sched"], r["bytes"])][proto] = (r["us"], mb)
    return pts


def fit(pts, proto):
    rows, y = [], []
    for (s, _), d in pts.items():
        if proto in d:
            us, mb = d[proto]
            rows.append([1.0 / us, STEPS[s] / us, mb / us])  # relative error: (model - us) / us
            y.append(1.0)
    sol, *_ = np.linalg.lstsq(np.array(rows), np.array(y), rcond=None)
    return sol


def regret(pts, co):
    regrets = []
    for (s, sz), d in sorted(pts.items()):
        if len(d) < 2:
            continue
        pred = {p: co[p][0] + co[p][1] * STEPS[s] + co[p][2] * d[p][1] for p in d}
        pick = min(pred, key=pred.get)
        best = min(v[0] for v in d.values())
        regrets.append((d[pick][0] / best - 1, s, sz, pick))
    return regrets


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--eval")]
    ev = [a.split("=", 1)[1] if "=" in a else None for a in sys.argv[1:] if a.startswith("--eval")]
    if "--eval" in sys.argv:
        i = sys.argv.index("--eval")
        ev = [sys.argv[i + 1]]
        args = [a for j, a in enumerate(sys.argv[1:], 1) if j not in (i, i + 1)]
    pts = load(args)
    if ev and ev[0]:
        v = [float(x) for x in ev[0].split(",")]
        r = regret(pts, {"ll": v[:3], "simple": v[3:]})
        a = np.array([x[0] for x in r])
        print(f"given constants: points {len(a)}  mean regret {100 * a.mean():.1f} %  worst {100 * a.max():.1f} % "
              f"({max(r)[1]} {max(r)[2]})")
    co = {p: fit(pts, p) for p in ("ll", "simple")}
    for p, (c, a, b) in co.items():
        print(f"{p:6s} c={c:.2f} us  a={a:.3f} us/step  b={b:.4f} us/MB")
    regrets = []
    for (s, sz), d in sorted(pts.items()):
        if len(d) < 2:
            continue
        # the MB a protocol's program moves differs (LL slots are 2x): predict each with its own MB
        pred = {p: co[p][0] + co[p][1] * STEPS[s] + co[p][2] * d[p][1] for p in d}
        pick = min(pred, key=pred.get)
        best = min(v[0] for v in d.values())
        regrets.append((d[pick][0] / best - 1, s, sz, pick))
    r = np.array([x[0] for x in regrets])
    print(f"points {len(r)}  mean regret {100 * r.mean():.1f} %  worst {100 * r.max():.1f} % "
          f"({max(regrets)[1]} {max(regrets)[2]})")
    print(json.dumps({p: [round(float(v), 4) for v in co[p]] for p in co}))


if __name__ == "__main__":
    main()
