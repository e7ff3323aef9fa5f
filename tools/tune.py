#!/usr/bin/env python3
"""Loopback tuning matrix on one GPU: for each (schedule, size, knob set)
time the executor (CUDA events) and print one JSON line.  Knobs: tile,
stage budget (env SCCL_STAGE_BUDGET), chunk groups, byte parts, protocol,
and "env": any SCCL_* plan variable set for that plan only."""
import itertools
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2008_08708_b200 import sccl  # noqa: E402
from paper_2008_08708_b200 import schedules as S  # noqa: E402


def time_plan(plan, send, recv, iters):
    st = torch.cuda.Stream()
    torch.cuda.synchronize()  # inputs may come from the default stream
    for _ in range(3):
        plan.launch(send, recv, st)
    st.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for _ in range(iters):
            plan.launch(send, recv, st)
    with torch.cuda.stream(st):  # replay() launches on the current stream
        g.replay()
        st.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        g.replay()
        b.record(st)
    st.synchronize()
    plan.check()
    return a.elapsed_time(b) * 1e3 / iters


def cudart():
    import ctypes
    import glob
    import nvidia.cuda_runtime as m
    return ctypes.CDLL(glob.glob(os.path.join(m.__path__[0], "lib", "libcudart.so*"))[0])


def set_persisting_l2(nbytes):
    """cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize): the L2 set-aside
    that evict_last accesses may occupy."""
    import ctypes
    rt = cudart()
    rc = rt.cudaDeviceSetLimit(ctypes.c_int(0x06), ctypes.c_size_t(nbytes))
    v = ctypes.c_size_t(0)
    rt.cudaDeviceGetLimit(ctypes.byref(v), ctypes.c_int(0x06))
    mx = ctypes.c_int(0)
    rt.cudaDeviceGetAttribute(ctypes.byref(mx), ctypes.c_int(108), ctypes.c_int(0))
    return rc, v.value, mx.value


def main():
    P = 8
    ag = S.hamiltonian_allgather(P)
    scheds = {"ag777": (S.to_json(ag), sccl.U8), "ag111": (S.to_json(S.one_shot_allgather(P)), sccl.U8),
              "ar822": (S.allreduce_from(S.one_shot_allgather(P)), sccl.BF16),
              "ar56": (S.allreduce_from(ag), sccl.BF16),
              "ring": (S.to_json(S.ring_allgather(P)), sccl.U8),
              "ar_ring": (S.allreduce_from(S.ring_allgather(P)), sccl.BF16),
              "a2a": (S.to_json(S.direct_alltoall(P)), sccl.U8),
              # floor: one rank, no sends (launch + prologue + a local copy)
              "null1": (S.to_json(S._sched("allgather", "full:1", 1, 1, 1, [1], [])), sccl.U8)}
    grid = json.loads(sys.argv[1]) if len(sys.argv) > 1 else {}
    sizes = grid.get("sizes", [128 << 20])
    names = grid.get("scheds", list(scheds))
    knobs = grid.get("knobs", [{}])
    maxb = max(sizes)
    send = [torch.randint(0, 256, (maxb,), dtype=torch.uint8, device="cuda") for _ in range(P)]
    recv = [torch.empty(P * maxb, dtype=torch.uint8, device="cuda") for _ in range(P)]
    for name, sz, kn in itertools.product(names, sizes, knobs):
        js, dt = scheds[name]
        if "order" in kn:
            os.environ["SCCL_SEND_ORDER"] = kn["order"]
        else:
            os.environ.pop("SCCL_SEND_ORDER", None)
        persist = set_persisting_l2(kn.get("persist", 0))
        for k, v in kn.get("env", {}).items():  # e.g. {"SCCL_WINDOW": "32768"}: read at plan creation
            os.environ[k] = str(v)
        if "budget" in kn:
            os.environ["SCCL_STAGE_BUDGET"] = str(kn["budget"])
        else:
            os.environ.pop("SCCL_STAGE_BUDGET", None)
        try:
            plan = sccl.LoopbackPlan(js, sz, dt, device=0, nchannels=kn.get("kb", 0), chunk_groups=kn.get("kc", 0),
                                     tile_bytes=kn.get("tile", 0), protocol=kn.get("protocol", "auto"),
                                     pull=kn.get("pull", "auto"))
        except sccl.SCCLError as e:
            print(json.dumps({"sched": name, "bytes": sz, "knobs": kn, "error": str(e)[:100]}), flush=True)
            continue
        for k in kn.get("env", {}):
            os.environ.pop(k, None)
        rb = plan.recv_bytes
        us = time_plan(plan, [x[:sz] for x in send], [x[:rb] for x in recv], 20 if sz >= (16 << 20) else 100)
        info = plan.info()
        prog = info["program"]
        hbm = sum(op["len"] * (len(op["ins"]) + len(op["outs"])) for rk in prog["ranks"] for op in rk["ops"]
                  if op["kind"] != "wait")
        print(json.dumps({"sched": name, "bytes": sz, "knobs": kn, "us": round(us, 2),
                          "hbm_TBps": round(hbm / us / 1e6, 3), "kc": info["chunk_groups"], "kb": info["byte_parts"],
                          "tile": info["tile_bytes"], "nstage": info["nstage"], "proto": info["protocol"],
                          "grid": info["grid"], "window": info["window"], "pull": info["pull"],
                          "persist_l2": persist}), flush=True)
        plan.close()


def main_multi(grid):
    """--multi: the N>1 refit (run under torchrun, one rank per GPU).  Times
    every (schedule, size, protocol, nchannels) of the grid with one rank
    per GPU (CUDA events, max over ranks), refits the protocol model
    c + alpha * steps + beta * MB (this rank's program bytes) per protocol by
    relative-error least squares, picks the CTAs-per-rank cap that wins most
    often, and writes a policy table for SCCL_POLICY (the "multiprocess"
    section of policy.hpp's ModePolicy) to grid["out"]."""
    import time
    import numpy as np
    import torch.distributed as dist
    rank, P = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    shared = os.environ.get("SCCL_BENCH_SHARE_GPU") == "1"
    dev = 0 if shared else int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(dev)
    if shared:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
    bench_dir = os.path.join(ROOT, "tests", "golden", "schedules", "bench")
    names = grid.get("scheds", [f"ag_oneshot_full{P}", f"ag_ring_ring{P}", f"ar_oneshot_full{P}",
                                f"ar_ring_ring{P}", f"a2a_direct_full{P}"])
    sizes = grid.get("sizes", [1 << k for k in range(10, 27, 2)])
    chans = grid.get("nchannels", [0])
    maxb = max(sizes)
    send = torch.randint(0, 256, (maxb,), dtype=torch.uint8, device="cuda")
    rows = []
    for name in names:
        js = open(os.path.join(bench_dir, name + ".json")).read()
        d = json.loads(js)
        steps = sum(ph["S"] for ph in d.get("phases", [d]))
        dt = sccl.BF16 if d["collective"] == "allreduce" else sccl.U8
        for sz, proto, nch in itertools.product(sizes, ("ll", "simple"), chans):
            if d["collective"] == "alltoall" and sz % (P * 2):
                continue
            plan = sccl.Plan(js, rank, P, sz, dt, device=dev, protocol=proto, nchannels=nch)
            plan.bind_with()
            reg, _ = plan.recv_buffer()
            s = send[:plan.send_bytes]
            iters = 50 if sz <= (1 << 20) else 10
            for _ in range(3):
                plan.launch(s, reg)
            dist.barrier()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(iters):
                plan.launch(s, reg)
            b.record()
            torch.cuda.synchronize()
            t = torch.tensor([a.elapsed_time(b) * 1e3 / iters], device="cpu" if shared else "cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            info = plan.info()
            mb = sum(op["len"] * (len(op["ins"]) + len(op["outs"])) for op in info["program"]["ranks"][rank]["ops"]
                     if op["kind"] != "wait") / 1e6
            r = {"sched": name, "steps": steps, "bytes": sz, "protocol": proto, "nchannels": info["nchannels"],
                 "us": round(float(t), 2), "mb": mb}
            rows.append(r)
            if rank == 0:
                print(json.dumps(r), flush=True)
            plan.close()
    if rank == 0:
        co = {}
        for proto in ("ll", "simple"):
            pts = [r for r in rows if r["protocol"] == proto]
            A = np.array([[1.0 / r["us"], r["steps"] / r["us"], r["mb"] / r["us"]] for r in pts])
            try:  # the constants are times: non-negative least squares
                from scipy.optimize import nnls
                sol, _ = nnls(A, np.ones(len(pts)))
            except ImportError:
                sol, *_ = np.linalg.lstsq(A, np.ones(len(pts)), rcond=None)
            co[proto] = [round(float(x), 4) for x in sol]
        wins = {}
        for key in {(r["sched"], r["bytes"]) for r in rows}:
            best = min((r for r in rows if (r["sched"], r["bytes"]) == key), key=lambda r: r["us"])
            wins[best["nchannels"]] = wins.get(best["nchannels"], 0) + 1
        table = {"multiprocess": {
            "version": f"multiprocess-nvlink-P{P}-{time.strftime('%Y%m%d')}",
            "ll_c": co["ll"][0], "ll_alpha": co["ll"][1], "ll_beta": co["ll"][2],
            "simple_c": co["simple"][0], "simple_alpha": co["simple"][1], "simple_beta": co["simple"][2],
            "max_ctas_per_rank": max(wins, key=wins.get) if len(chans) > 1 else 32}}
        out = grid.get("out", os.path.join(ROOT, "gpurun_out", f"policy_multiprocess_P{P}.json"))
        with open(out, "w") as f:
            json.dump(table, f, indent=1)
        print(json.dumps({"policy_table": out, **table}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--multi":
        main_multi(json.loads(sys.argv[2]) if len(sys.argv) > 2 else {})
    else:
        main()
