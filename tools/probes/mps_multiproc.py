#!/usr/bin/env python3
"""The one-rank-per-process path timed with every rank running CONCURRENTLY
on one GPU under MPS (run under torchrun with CUDA_MPS_PIPE_DIRECTORY set
and the MPS daemon started; gloo): CUDA IPC peers, system-scope counters,
entry handshakes / parity slot sets, one launch per rank -- the N>1 kernel
path with its HBM shared instead of NVLink between the ranks.  For each
(schedule, size, protocol, variant) it prints the max-over-ranks time per
launch of `iters` back-to-back launches (CUDA events, after a barrier) and
checks the last output against the oracle.
usage: torchrun --nproc-per-node 8 tools/probes/mps_multiproc.py"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import oracle as O  # noqa: E402
from paper_2008_08708_b200 import sccl  # noqa: E402

SCHED_DIR = os.path.join(ROOT, "tests", "golden", "schedules", "bench")


def main():
    dist.init_process_group("gloo")
    rank, W = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    cases = []
    for name, dt in ((f"ag_oneshot_full{W}", O.U8), (f"ag_ring_ring{W}", O.U8), (f"ar_oneshot_full{W}", O.BF16),
                     (f"a2a_direct_full{W}", O.U8)):
        for nb in (1024, 16384, 65536):
            cases.append((name, dt, nb, "ll", "1"))
            cases.append((name, dt, nb, "ll", "0"))
        for nb in (1 << 20, 16 << 20, 64 << 20):
            cases.append((name, dt, nb, "simple", "1"))
    if W == 8:
        cases += [(f"ag_ham_full{W}", O.U8, 128 << 20, "simple", "1"), (f"ar_ham_full{W}", O.BF16, 64 << 20, "simple", "1")]
    for name, dt, nb, proto, parity in cases:
        js = open(os.path.join(SCHED_DIR, name + ".json")).read()
        d = json.loads(js)
        if d["collective"] == "alltoall" and nb % W:
            continue
        os.environ["SCCL_LL_PARITY"] = parity
        # every rank's CTAs share one GPU here: simple plans get 16 CTAs per
        # rank so that W x 16 fit even where the policy picks 1 CTA per SM
        # (wide reductions) -- one rank per GPU needs no such cap
        nch = 16 if (proto == "simple" and W * 32 > 148) else 0
        plan = sccl.Plan(js, rank, W, nb, dt, device=0, protocol=proto, timeout_ms=60000, nchannels=nch)
        os.environ.pop("SCCL_LL_PARITY")
        plan.bind_with()
        ins = O.seeded_inputs(d["collective"], W, nb, dt, 7)
        want = O.execute(d, ins, nb, dt)[rank]
        send = torch.from_numpy(ins[rank]).cuda()
        reg, _ = plan.recv_buffer()
        iters = 200 if nb <= (1 << 20) else 20
        for _ in range(3):
            plan.launch(send, reg)
        torch.cuda.synchronize()
        dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(iters):
            plan.launch(send, reg)
        b.record()
        torch.cuda.synchronize()
        plan.check()
        t = torch.tensor([a.elapsed_time(b) * 1e3 / iters])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        out = torch.empty(want.size, dtype=torch.uint8, device="cuda")
        plan.launch(send, out)
        torch.cuda.synchronize()
        ok = [None] * W
        dist.all_gather_object(ok, bool(np.array_equal(out.cpu().numpy(), want)))
        if rank == 0:
            print(json.dumps({"schedule": name, "bytes_per_rank": nb, "protocol": proto,
                              "ll_parity": plan.info()["ll_parity"], "nchannels": plan.info()["nchannels"],
                              "us": round(float(t), 2), "ranks_exact": all(ok)}), flush=True)
        dist.barrier()
        plan.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
