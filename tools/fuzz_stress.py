#!/usr/bin/env python3
"""GPU stress fuzzer: random valid schedules (tests/test_fuzz.py's
generator) x random plan modes -- protocol, chunk groups / byte parts,
counter-release mode, window-major byte window, L2 hints, receipt discards
(forced through the SCCL_* variables, read at plan creation) -- each launched
twice and compared bit for bit with the oracle.  One JSON summary line;
failing cases are listed with everything needed to replay them.

usage: python tools/fuzz_stress.py [ncases] [seed]"""
import json
import os
import random
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
from paper_2008_08708_b200 import sccl  # noqa: E402
from paper_2008_08708_b200 import schedules as S  # noqa: E402

ENV = ("SCCL_WINDOW", "SCCL_L2HINT", "SCCL_DISCARD", "SCCL_SELFPUB")


def case(rng, i, seed):
    P = rng.choice([2, 3, 4, 5, 6, 8])
    C = rng.choice([1, 2, 3])
    St = rng.randint(1, 4)
    ag = sccl.canonicalize(json.dumps(S.random_allgather(P, C, St, seed=seed * 100000 + i)))
    kind = rng.choice(["ag", "rs", "ar"])
    js = ag if kind == "ag" else sccl.invert(ag) if kind == "rs" else sccl.compose_allreduce(sccl.invert(ag), ag)
    dt = O.U8 if kind == "ag" else rng.choice([O.I32, O.F32, O.BF16, O.F16])
    nb = rng.choice([16, 4096, 12000 + 16 * rng.randint(0, 100), 1 << 18, (1 << 20) + 48, 3 << 20])
    nb -= nb % O.ESIZE[dt]
    mode = {"protocol": rng.choice(["ll", "simple", "simple", "auto"]),
            "kc_kb": rng.choice([(0, 0), (0, 0), (2, 3), (1, 1), (3, 2)]),
            "env": {"SCCL_WINDOW": rng.choice(["0", "4096", "65536", None]),
                    "SCCL_L2HINT": rng.choice(["0", "1", None]),
                    "SCCL_DISCARD": rng.choice(["0", "1", None]),
                    "SCCL_SELFPUB": rng.choice(["0", "1", None])}}
    return js, nb, dt, mode


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 300
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 7
    rng = random.Random(seed)
    fails, t0, done = [], time.time(), 0
    for i in range(n):
        js, nb, dt, mode = case(rng, i, seed)
        for k in ENV:
            v = mode["env"][k]
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
        d = json.loads(js)
        ins = O.seeded_inputs(d["collective"], d["P"], nb, dt, i)
        ref = O.execute(d, ins, nb, dt)
        kc, kb = mode["kc_kb"]
        try:
            plan = sccl.LoopbackPlan(js, nb, dt, device=0, protocol=mode["protocol"], chunk_groups=kc, nchannels=kb,
                                     timeout_ms=20000)
        except sccl.SCCLError as e:  # e.g. a channel request over the resident-CTA limit
            if "resident" in str(e) or "channels" in str(e):
                continue
            raise
        send = [torch.from_numpy(x).cuda() for x in ins]
        recv = [torch.zeros(r.size, dtype=torch.uint8, device="cuda") for r in ref]
        torch.cuda.synchronize()
        for _ in range(2):
            plan.launch(send, recv)
        torch.cuda.synchronize()
        plan.check()
        bad = [r for r, (a, b) in enumerate(zip(recv, ref)) if not np.array_equal(a.cpu().numpy(), b)]
        if bad:
            fails.append({"case": i, "seed": seed, "kind": d["collective"], "P": d["P"], "bytes": nb, "dtype": dt,
                          "mode": mode, "ranks": bad, "info": {k: plan.info()[k] for k in
                                                               ("protocol", "window", "selfpub", "l2hint", "discard",
                                                                "chunk_groups", "byte_parts", "tile_bytes")}})
        plan.close()
        done += 1
    for k in ENV:
        os.environ.pop(k, None)
    print(json.dumps({"cases": done, "failures": len(fails), "seconds": round(time.time() - t0, 1),
                      "failed": fails[:20]}))


if __name__ == "__main__":
    main()
