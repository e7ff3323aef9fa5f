#!/usr/bin/env python3
"""Multi-process fuzzer: random valid schedules for P = WORLD_SIZE ranks
(tests/test_fuzz.py's generator; allgather, its inverted reduce-scatter and
the composed allreduce) x random plan modes (protocol, chunk groups / byte
parts, LL parity on/off, counter-release mode), executed on the
one-rank-per-process path -- IPC-mapped peers, sys-scope counters, entry
handshake or parity slots -- with every rank in its own process (gloo; all
on cuda:0 unless LOCAL_RANK devices exist and SCCL_FUZZ_DEVICES=1).  Each
case launches twice back to back (no barrier between) and every rank
compares both outputs with the oracle.  Every rank draws the same cases
from the same seed.  Rank 0 prints one JSON summary line.

usage: torchrun --nproc-per-node W tools/fuzz_multiproc.py [ncases] [seed]"""
import json
import os
import random
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import oracle as O  # noqa: E402
from paper_2008_08708_b200 import sccl  # noqa: E402
from paper_2008_08708_b200 import schedules as S  # noqa: E402


def case(rng, P, i, seed):
    C = rng.choice([1, 2, 3])
    St = rng.randint(1, 4)
    ag = sccl.canonicalize(json.dumps(S.random_allgather(P, C, St, seed=seed * 100000 + i)))
    kind = rng.choice(["ag", "rs", "ar"])
    js = ag if kind == "ag" else sccl.invert(ag) if kind == "rs" else sccl.compose_allreduce(sccl.invert(ag), ag)
    dt = O.U8 if kind == "ag" else rng.choice([O.I32, O.F32, O.BF16, O.F16])
    nb = rng.choice([16, 4096, 12000 + 16 * rng.randint(0, 100), 1 << 17, (1 << 18) + 48])
    nb -= nb % O.ESIZE[dt]
    mode = {"protocol": rng.choice(["ll", "simple", "auto"]),
            "nch": rng.choice([0, 0, 1, 3, 8]),
            "kc": rng.choice([0, 0, 1, 2]),
            "parity": rng.choice(["1", "0"]),
            "selfpub": rng.choice(["0", "1", None])}
    return js, nb, dt, mode


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 50
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 11
    dist.init_process_group("gloo")
    rank, P = dist.get_rank(), dist.get_world_size()
    dev = int(os.environ.get("LOCAL_RANK", rank)) if os.environ.get("SCCL_FUZZ_DEVICES") == "1" else 0
    torch.cuda.set_device(dev)
    rng = random.Random(seed)
    fails, t0 = [], time.time()
    for i in range(n):
        js, nb, dt, mode = case(rng, P, i, seed)
        os.environ["SCCL_LL_PARITY"] = mode["parity"]
        if mode["selfpub"] is None:
            os.environ.pop("SCCL_SELFPUB", None)
        else:
            os.environ["SCCL_SELFPUB"] = mode["selfpub"]
        d = json.loads(js)
        err = None
        try:
            plan = sccl.Plan(js, rank, P, nb, dt, device=dev, protocol=mode["protocol"], nchannels=mode["nch"],
                             chunk_groups=mode["kc"], timeout_ms=60000)
            try:
                plan.bind_with()
                outs = []
                for it in range(2):  # back to back, no barrier between the launches
                    ins = O.seeded_inputs(d["collective"], P, nb, dt, 1000 * i + it)
                    want = O.execute(d, ins, nb, dt)[rank]
                    recv = torch.full((max(want.size, 1),), 0xEE, dtype=torch.uint8, device=f"cuda:{dev}")
                    plan.launch(torch.from_numpy(ins[rank]).to(recv.device), recv)
                    outs.append((recv, want))
                torch.cuda.synchronize()
                plan.check()
                for it, (recv, want) in enumerate(outs):
                    if not np.array_equal(recv.cpu().numpy()[:want.size], want):
                        err = f"launch {it} differs from the oracle"
            finally:
                plan.close()
        except Exception as e:  # noqa: BLE001 -- reported
            err = f"{type(e).__name__}: {e}"[:300]
        errs = [None] * P
        dist.all_gather_object(errs, err)
        if any(errs):
            fails.append({"case": i, "schedule": d["collective"], "C": d.get("C"), "S": d.get("S"), "bytes": nb,
                          "dtype": dt, "mode": mode, "errors": {r: e for r, e in enumerate(errs) if e}})
        dist.barrier()
    if rank == 0:
        print(json.dumps({"ranks": P, "cases": n, "failures": len(fails), "seconds": round(time.time() - t0, 1),
                          "failed": fails[:10]}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
