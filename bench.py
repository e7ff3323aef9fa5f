#!/usr/bin/env python3
"""Benchmark: collective bus GB/s of the B200 executor for SCCL-synthesized
schedules (BASELINE.json metric), with the CPU reference executor and (N>1)
NCCL beside it.

Metric convention (nccl-tests busBW): bus GB/s per rank =
algorithmic bytes each rank sends per launch / time; allgather (P-1)*m.
`value` is that per-rank figure summed over the GPUs of the job:
  N = 1   the BASELINE config 2 allgather (C,S,R) = (7,7,7) on full(8) with
          all 8 ranks in LOOPBACK on cuda:0 (one launch runs every rank's
          channel program; all rank buffers in one HBM), 128 MiB per rank.
          One GPU => value = the per-rank bus bandwidth (the 8-rank sum is
          reported beside it as aggregate_GBps), so a 1/2/4/8-GPU series
          compares per-rank collective speed.
  N > 1   (torchrun) one rank per GPU, peers' plan regions mapped through
          CUDA IPC over NVLink/NVSwitch; value = N * per-rank bus GB/s.
          NCCL is timed on the same buffers (allgather default and
          NCCL_PROTO=Simple, allreduce Ring/Tree, alltoall as grouped
          send/recv), plus a <= 64 KB latency sweep and NVML NVLink byte
          counters around the timed region.
e2e: the same metric through the public API with host buffers, every step:
          H2D of every rank's input, the collective, D2H of every rank's
          whole output.
--impl reference: the CPU reference executor (oracle/: the C restatement of
          SPEC.md:418-426, pthreads on all host cores) on the GPU arm's exact
          workload (same schedule file, ranks, bytes per rank).  It imports
          nothing from the product package: the schedule comes from the
          committed file tests/golden/schedules/bench/*.json.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
SCHED_DIR = os.path.join(ROOT, "tests", "golden", "schedules", "bench")
sys.path.insert(0, ROOT)

METRIC = "collective bus GB/s and latency vs buffer size at 2/4/8 B200 vs NCCL and CPU ref"
NVLINK_PEAK = 900.0  # GB/s per direction per GPU, NVLink 5 (nominal)
# N > 1: peer-wait watchdog of every bench plan (the library default for one
# rank per GPU is 600 s); every launch here takes milliseconds, so a peer that
# has not signalled within a minute is a failure the line should report
BENCH_TIMEOUT_MS = 60000
# N > 1: the comparison sections (NCCL, NVLS, sweep) start only while the run
# is younger than this; the line says which were skipped
EXTRAS_BUDGET_S = float(os.environ.get("SCCL_BENCH_EXTRAS_S", "420"))


def load_schedule(name: str) -> str:
    with open(os.path.join(SCHED_DIR, name + ".json")) as f:
        return f.read().strip()


def sched_label(name: str) -> str:
    d = json.loads(load_schedule(name))
    return f"{d['collective']} ({d['C']},{d['S']},{d['R']}) {name}, {d['topology']['name']}"


def workload_schedule(P: int, which: str) -> str:
    """bench schedule file for the allgather workload at P ranks"""
    if which == "auto":
        which = "ham" if P in (2, 8) else "oneshot"
    if P == 1:  # the multi-process path's one-GPU self-test (SCCL_BENCH_FORCE_MULTI=1)
        which = "oneshot"
    return {"ham": f"ag_ham_full{P}", "oneshot": f"ag_oneshot_full{P}", "ring": f"ag_ring_ring{P}"}[which]


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return {"hbm_gbs": 6650.0}, "fallback (B200_PROFILING.md)"


def _profile_traffic(key: str):
    """ncu dram__bytes_read+write per launch recorded for this workload by a
    committed profile (profiles/traffic.json: key -> {bytes, source})."""
    try:
        t = json.load(open(os.path.join(ROOT, "profiles", "traffic.json"))).get(key)
    except Exception:
        return None, None
    if isinstance(t, dict):
        return t.get("bytes"), t.get("source")
    return t, "profiles/traffic.json"


class ClockSampler:
    """SM clocks, board power and throttle reasons sampled during the timed
    region (NVML in-process; nvidia-smi if NVML is unavailable)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int = 0):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _nvml_handle(self):
        """In-process NVML (the device matched by PCI bus id), sampled every
        50 ms: more samples than one nvidia-smi process per 0.2 s, plus the
        board power.  (The two samplers time the bench workload alike:
        tools/gpu_runs/r02/s2_sampler_ab.sh.)"""
        if os.environ.get("SCCL_BENCH_SMI") == "1":  # A/B: the subprocess sampler
            return None, None
        try:
            import pynvml
            import torch
            pynvml.nvmlInit()
            pr = torch.cuda.get_device_properties(self.index)
            bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
            try:
                return pynvml, pynvml.nvmlDeviceGetHandleByPciBusId(bus.encode())
            except Exception:
                return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.index)
        except Exception:
            return None, None

    def _run(self):
        nv, h = self._nvml_handle()
        self.kind = "nvml" if h is not None else "nvidia-smi"
        if h is not None:
            bits = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                    "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                    "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap}
            while not self._stop.is_set():
                try:
                    sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                    mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
                    pw = nv.nvmlDeviceGetPowerUsage(h) / 1000.0
                    rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.rows.append([str(self.index), str(sm), str(mx), f"{pw:.1f}", hex(rs)] +
                                     ["Active" if rs & b else "Not Active" for b in bits.values()])
                except Exception:
                    pass
                self._stop.wait(0.05)
            return
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 5 + i and r[5 + i] == "Active"})
        pw = [float(r[3]) for r in self.rows if r[3].replace(".", "").isdigit()]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows), "power_w_max": max(pw) if pw else None,
                "sampler": getattr(self, "kind", None)}


def busbytes(coll: str, P: int, m: int) -> int:
    """bytes each rank sends per launch (nccl-tests busBW numerator)"""
    if coll == "allgather":
        return (P - 1) * m
    if coll == "allreduce":
        return 2 * (P - 1) * m // P
    return (P - 1) * m // P  # alltoall, reducescatter


def hbm_bytes_per_launch(plan) -> int:
    """Bytes the lowered program reads and writes (every op's inputs and
    outputs once; loopback: the whole launch)."""
    info = plan.info()["program"]
    return sum(op["len"] * (len(op["ins"]) + len(op["outs"])) for rk in info["ranks"] for op in rk["ops"]
               if op["kind"] != "wait")


def host_cpu() -> str:
    """CPU model and logical CPU count of the host the CPU baselines ran on
    (SURVEY.md 8(d) cfg 1: record the GPU box's CPU)."""
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return f"{model}, {os.cpu_count()} logical CPUs"


def _oracle():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    return O


# --------------------------------------------------------------------------- reference arm (CPU)
def run_reference(args):
    """The reference's own executor (restated in C under
    oracle/) on the host cores, on the GPU arm's workload.  Rank 0 only."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    P = 8 if args.gpus == 1 else args.gpus
    name = workload_schedule(P, args.schedule)
    js = load_schedule(name)
    m = args.ref_bytes if args.ref_bytes > 0 else args.bytes
    threads = os.cpu_count() or 1
    O = _oracle()
    d = json.loads(js)
    ins = O.seeded_inputs(d["collective"], P, m, O.U8, 0)
    ex = O.Execution(d, ins, m, O.U8, check=True)  # the oracle's own verify gate
    for _ in range(args.warmup):
        ex.run(threads)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        ex.run(threads)
        times.append(time.perf_counter() - t0)
    want = b"".join(x.tobytes() for x in ins)
    out = ex.outputs()
    assert out[0].tobytes() == want and out[P - 1].tobytes() == want, "reference executor result wrong"
    t = sum(times) / len(times)
    per_rank = busbytes("allgather", P, m) / t / 1e9
    value = per_rank * (1 if args.gpus == 1 else P)
    sample = (f"oracle executor loop (SPEC.md:418-426 restated in C, {threads} threads) on {P} ranks x {m} B per "
              f"rank, schedule file {name}.json; every step is one whole execution of the workload")
    line = {"metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(1e3 * t, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic (seeded PRNG bytes)",
            "impl": "reference",
            "config": {"workload": _workload_text(args.gpus, P, name), "ranks": P, "bytes_per_rank": m,
                       "schedule": sched_label(name), "schedule_file": f"tests/golden/schedules/bench/{name}.json",
                       "same_config": m == args.bytes, "executor": "CPU reference (oracle port)",
                       "parallelism": f"{threads} host threads"},
            "aggregate_GBps": round(per_rank * P, 3),
            "cpu_baseline": {"value": round(value, 3), "unit": "GB/s", "cores": threads, "kind": "port",
                             "sample": sample, "host_cpu": host_cpu()},
            "e2e": {"value": round(value, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _workload_text(gpus: int, P: int, name: str, multi: bool = False) -> str:
    if gpus == 1 and not multi:
        return f"{sched_label(name)}; {P} ranks loopback on 1 B200 (all rank buffers in one HBM)"
    return f"{sched_label(name)}; one rank per GPU on {P} B200s, CUDA IPC peers over NVLink/NVSwitch"


# --------------------------------------------------------------------------- GPU helpers
def graph_time_us(plan, send, recv, stream, iters, reps=3):
    """Device time per launch: `iters` launches captured in one CUDA graph
    (host launch cost excluded), replayed once untimed, then `reps` timed
    replays; the median replay (a single short replay of microsecond
    launches moved with the clock state the previous sweep point left)."""
    import torch
    for _ in range(3):
        plan.launch(send, recv, stream)
    stream.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for _ in range(iters):
            plan.launch(send, recv, stream)
    ts = []
    with torch.cuda.stream(stream):  # replay() launches on the current stream
        g.replay()
        stream.synchronize()
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            g.replay()
            b.record(stream)
            stream.synchronize()
            ts.append(a.elapsed_time(b) * 1e3 / iters)
    plan.check()
    return statistics.median(ts)


def oracle_check_loopback(sccl, name, nbytes, dtype, seed=5):
    """Bit-exact check of every rank's output against the CPU oracle on the
    same schedule file (small size); returns {rank: digest_equal}."""
    import numpy as np
    import torch
    O = _oracle()
    js = load_schedule(name)
    d = json.loads(js)
    P = d["P"]
    ins = O.seeded_inputs(d["collective"], P, nbytes, dtype, seed)
    ref = O.execute(d, ins, nbytes, dtype)
    plan = sccl.LoopbackPlan(js, nbytes, dtype, device=0)
    send = [torch.from_numpy(x).cuda() for x in ins]
    recv = [torch.zeros(r.size, dtype=torch.uint8, device="cuda") for r in ref]
    plan.launch(send, recv)
    torch.cuda.synchronize()
    plan.check()
    plan.close()
    return all(O.digest([a.cpu().numpy()]) == O.digest([b]) for a, b in zip(recv, ref))


# --------------------------------------------------------------------------- GPU, N = 1
def run_loopback(args):
    import torch
    from paper_2008_08708_b200 import sccl
    P = 8
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    name = workload_schedule(P, args.schedule)
    js = load_schedule(name)
    m = args.bytes
    plan = sccl.LoopbackPlan(js, m, sccl.U8, device=0, nchannels=args.nchannels, tile_bytes=args.tile)
    info = plan.info()
    send = [torch.randint(0, 256, (m,), dtype=torch.uint8, device=dev) for _ in range(P)]
    recv = [torch.empty(P * m, dtype=torch.uint8, device=dev) for _ in range(P)]
    stream = torch.cuda.Stream()
    torch.cuda.synchronize()  # inputs were generated on the default stream
    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            plan.launch(send, recv, stream)
    stream.synchronize()
    want = torch.cat(send)  # every rank holds the concatenation
    assert all(torch.equal(r, want) for r in recv), "bench: allgather result wrong"
    oracle_ok = oracle_check_loopback(sccl, name, 1 << 20, sccl.U8)

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    t_all = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
    torch.cuda.synchronize()
    with ClockSampler(0) as clk:
        t_soak = time.perf_counter()  # untimed soak so the clock record sees this load
        while time.perf_counter() - t_soak < 0.6:
            for _ in range(8):
                plan.launch(send, recv, stream)
            stream.synchronize()
        n0 = plan.launch_count
        t_all[0].record(stream)
        for i in range(args.steps):
            ev[i][0].record(stream)
            plan.launch(send, recv, stream)
            ev[i][1].record(stream)
        t_all[1].record(stream)
        torch.cuda.synchronize()
    launches = plan.launch_count - n0
    plan.check()
    ms = t_all[0].elapsed_time(t_all[1]) / args.steps
    kern_ms = sum(a.elapsed_time(b) for a, b in ev) / args.steps
    per_rank = busbytes("allgather", P, m) / (ms * 1e-3) / 1e9
    peaks, src = _peaks()
    sched_bytes = hbm_bytes_per_launch(plan)
    min_b = P * m + P * P * m  # inputs read once + outputs written once
    traffic, traffic_src = _profile_traffic(f"{name}:{m}")

    extra = {} if args.no_sweep else loopback_extras(args, sccl, plan, send, recv, stream, peaks)
    e2e = loopback_e2e(args, plan, send, recv)

    cpu_m = min(m, args.cpu_bytes)
    cpu_val, cpu_s, cpu_n = cpu_reference_run(P, js, cpu_m, args.cpu_seconds, 1)
    line = {
        "metric": METRIC, "value": round(per_rank, 2), "unit": "GB/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u8", "data": "synthetic (uniform random bytes)",
        "config": {"workload": _workload_text(1, P, name), "ranks": P, "bytes_per_rank": m,
                   "schedule": sched_label(name), "schedule_file": f"tests/golden/schedules/bench/{name}.json",
                   "nchannels": info["nchannels"], "tile_bytes": info["tile_bytes"], "grid": info["grid"],
                   "threads": info["threads"],
                   "l2": f"no flush: inputs {P * m >> 20} MiB + outputs {P * P * m >> 20} MiB per step >> 126 MB L2",
                   "parallelism": "loopback8",
                   "value_convention": "per-rank bus GB/s (nccl-tests busBW, (P-1)*m/t); one GPU"},
        "aggregate_GBps": round(per_rank * P, 2),
        "oracle_check": {"bytes_per_rank": 1 << 20, "all_ranks_bit_exact": oracle_ok},
        # algorithmic bytes = what any executor must move in one HBM: every
        # rank's input read once, every rank's output written once.  The
        # lowered (7,7,7) schedule also re-reads each relayed receipt to
        # forward it (schedule_bytes); window-major execution serves most of
        # those from L2, so ncu DRAM bytes land near the algorithmic bytes.
        "roofline": {"bound": "hbm", "achieved": round(min_b / (kern_ms * 1e-3) / 1e9, 1), "peak": peaks["hbm_gbs"],
                     "unit": "GB/s", "frac": round(min_b / (kern_ms * 1e-3) / 1e9 / peaks["hbm_gbs"], 4),
                     "traffic": traffic, "traffic_source": traffic_src, "peak_source": src,
                     "algorithmic_bytes_per_launch": min_b, "kernel_ms": round(kern_ms, 4),
                     "schedule_bytes_per_launch": sched_bytes,
                     "frac_schedule_bytes": round(sched_bytes / (kern_ms * 1e-3) / 1e9 / peaks["hbm_gbs"], 4)},
        "cpu_baseline": {"value": round(cpu_val / P, 3), "unit": "GB/s", "cores": 1, "kind": "port",
                         "sample": f"oracle executor, same schedule file, {P} ranks x {cpu_m} B, {cpu_n} runs in "
                                   f"{cpu_s:.1f} s, 1 thread (SPEC.md:447); per-rank bus GB/s",
                         "host_cpu": host_cpu()},
        "e2e": e2e,
        "clocks": clk.summary(),
        "gpu_launches": launches,
    }
    line.update(extra)
    print(json.dumps(line), flush=True)


def loopback_e2e(args, plan, send, recv):
    """Through the public API with host buffers, every step: H2D of all P
    ranks' inputs from pinned memory, the collective, D2H of ALL P ranks'
    outputs (P*P*m bytes).  Two device buffer sets and three streams overlap
    step i+1's H2D with step i's D2H; the timed region covers every step."""
    import torch
    P, m = len(send), send[0].numel()
    hsend = [[torch.empty(m, dtype=torch.uint8, pin_memory=True) for _ in range(P)] for _ in range(2)]
    for k in range(2):
        for h, x in zip(hsend[k], send):
            h.copy_(x.cpu())
    hres = torch.empty(P * P * m, dtype=torch.uint8, pin_memory=True)  # every rank's output
    dsend = [send, [torch.empty_like(x) for x in send]]
    drecv = [recv, [torch.empty_like(x) for x in recv]]
    s_h2d, s_k, s_d2h = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    steps = max(4, min(args.steps, 8))

    def run(nsteps):
        ev_in = [torch.cuda.Event() for _ in range(nsteps)]
        ev_k = [torch.cuda.Event() for _ in range(nsteps)]
        ev_out = [torch.cuda.Event() for _ in range(nsteps)]
        for i in range(nsteps):
            k = i % 2
            if i >= 2:  # buffer set k free: kernel(i-2) read its inputs, D2H(i-2) read its outputs
                s_h2d.wait_event(ev_k[i - 2])
            with torch.cuda.stream(s_h2d):
                for h, x in zip(hsend[k], dsend[k]):
                    x.copy_(h, non_blocking=True)
                ev_in[i].record(s_h2d)
            s_k.wait_event(ev_in[i])
            if i >= 2:
                s_k.wait_event(ev_out[i - 2])
            plan.launch(dsend[k], drecv[k], s_k)
            ev_k[i].record(s_k)
            s_d2h.wait_event(ev_k[i])
            with torch.cuda.stream(s_d2h):
                for r in range(P):
                    hres[r * P * m:(r + 1) * P * m].copy_(drecv[k][r], non_blocking=True)
                ev_out[i].record(s_d2h)
        return ev_out[-1]

    run(2)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s_h2d)
    s_k.wait_event(a)
    s_d2h.wait_event(a)
    last = run(steps)
    s_h2d.wait_event(last)
    b.record(s_h2d)
    torch.cuda.synchronize()
    e2e_ms = a.elapsed_time(b) / steps
    wc = torch.cat(hsend[0])  # both host input sets hold the same bytes
    assert all(torch.equal(hres[r * P * m:(r + 1) * P * m], wc) for r in range(P)), "e2e result wrong"

    # context, not the headline: one rank's share of the host traffic (its
    # input H2D, its output D2H) per step -- what each GPU of a one-rank-per-
    # GPU box moves over its own PCIe link; here all 8 ranks share one link
    def run_one(nsteps):
        ev_k = [torch.cuda.Event() for _ in range(nsteps)]
        for i in range(nsteps):
            k = i % 2
            with torch.cuda.stream(s_h2d):
                if i >= 2:
                    s_h2d.wait_event(ev_k[i - 2])
                dsend[k][0].copy_(hsend[k][0], non_blocking=True)
            s_k.wait_stream(s_h2d)
            s_k.wait_stream(s_d2h)
            plan.launch(dsend[k], drecv[k], s_k)
            ev_k[i].record(s_k)
            s_d2h.wait_event(ev_k[i])
            with torch.cuda.stream(s_d2h):
                hres[:P * m].copy_(drecv[k][0], non_blocking=True)
        return s_d2h

    run_one(2)
    torch.cuda.synchronize()
    a1, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a1.record(s_h2d)
    s_k.wait_event(a1)
    s_d2h.wait_event(a1)
    run_one(steps)
    b1.record(s_d2h)
    torch.cuda.synchronize()
    one_ms = a1.elapsed_time(b1) / steps
    return {"value": round(busbytes("allgather", P, m) / (e2e_ms * 1e-3) / 1e9, 3), "unit": "GB/s",
            "h2d_bytes_per_step": P * m, "d2h_bytes_per_step": P * P * m, "ms_per_step": round(e2e_ms, 3),
            "note": "per-rank bus GB/s through LoopbackPlan.launch with host buffers: H2D of all ranks' inputs + "
                    "collective + D2H of all ranks' outputs (8 GiB) every step, over one PCIe link; "
                    "pipelined over 2 device buffer sets / 3 streams",
            "per_gpu_pcie_variant": {
                "value": round(busbytes("allgather", P, m) / (one_ms * 1e-3) / 1e9, 3), "unit": "GB/s",
                "h2d_bytes_per_step": m, "d2h_bytes_per_step": P * m, "ms_per_step": round(one_ms, 3),
                "note": "context only: one rank's H2D + D2H per step (what each GPU of an 8-GPU box moves over "
                        "its own link); the headline e2e above copies every rank's data"}}


def loopback_extras(args, sccl, plan, send, recv, stream, peaks):
    """BASELINE configs 1, 3, 4 and the latency sweep on the same device."""
    import torch
    P = 8
    out = {}
    pk = peaks["hbm_gbs"]
    if send[0].numel() < (64 << 20):  # the sweeps below slice the workload's buffers
        return {"extras_skipped": "the config 1/3/4 sweeps need --bytes >= 64 MiB"}
    # latency sweep (CUDA-graph timed): allgathers, allreduces, alltoall
    sweep = []
    for sz in (1 << 10, 8 << 10, 64 << 10, 1 << 20, 16 << 20):
        row = {"bytes_per_rank": sz}
        for tag, nm, dt in (("ag777", "ag_ham_full8", sccl.U8), ("ag111", "ag_oneshot_full8", sccl.U8),
                            ("ar822_bf16", "ar_oneshot_full8", sccl.BF16), ("ar56_bf16", "ar_ham_full8", sccl.BF16),
                            ("a2a881", "a2a_direct_full8", sccl.U8)):
            p2 = sccl.LoopbackPlan(load_schedule(nm), sz, dt, device=0)
            coll = json.loads(load_schedule(nm))["collective"]
            us = graph_time_us(p2, [x[:p2.send_bytes] for x in send], [x[:p2.recv_bytes] for x in recv], stream,
                               200 if sz < (1 << 20) else 10)
            row[f"{tag}_us"] = round(us, 2)
            row[f"{tag}_busbw_per_rank_GBps"] = round(busbytes(coll, P, sz) / (us * 1e-6) / 1e9, 2)
            row[f"{tag}_protocol"] = p2.info()["protocol"]
            p2.close()
        sweep.append(row)
    out["latency_sweep"] = sweep

    # configs 3 and 4 at 64 MiB per rank (HBM floor = inputs once + outputs once)
    M = 64 << 20
    xs, ys = [x[:M] for x in send], [x[:M] for x in recv]
    oc = {}
    for tag, nm, dt in (("allreduce_56_14_14_bf16", "ar_ham_full8", sccl.BF16),
                        ("allreduce_56_14_14_f32", "ar_ham_full8", sccl.F32),
                        ("allreduce_8_2_2_bf16", "ar_oneshot_full8", sccl.BF16),
                        ("allreduce_8_2_2_f32", "ar_oneshot_full8", sccl.F32),
                        ("allreduce_ring_8_14_14_bf16", "ar_ring_ring8", sccl.BF16),
                        ("alltoall_8_1_1_u8", "a2a_direct_full8", sccl.U8)):
        p2 = sccl.LoopbackPlan(load_schedule(nm), M, dt, device=0)
        coll = json.loads(load_schedule(nm))["collective"]
        us = graph_time_us(p2, xs, ys, stream, 10)
        floor = 2 * P * M
        oc[tag] = {"bytes_per_rank": M, "us": round(us, 1),
                   "busbw_per_rank_GBps": round(busbytes(coll, P, M) / (us * 1e-6) / 1e9, 1),
                   "frac_of_hbm_floor": round(floor / (us * 1e-6) / 1e9 / pk, 3),
                   "schedule_bytes_GBps": round(hbm_bytes_per_launch(p2) / (us * 1e-6) / 1e9, 1),
                   "pull": p2.info()["pull"], "grid": p2.info()["grid"]}
        dram, dsrc = _profile_traffic(f"{nm}:{dt}:{M}")
        if dram:
            oc[tag]["dram_traffic"] = dram
            oc[tag]["dram_traffic_source"] = dsrc
        p2.close()
    out["other_collectives"] = oc
    out["allreduce_e2e"] = allreduce_e2e(sccl, xs, ys, stream)

    # config 1: ring(8) latency-optimal allgathers at 1 MiB per rank, the CPU
    # reference executor (1 thread and all threads) beside the GPU executor,
    # with the host memcpy roofline of the CPU side
    O = _oracle()
    c1 = {}
    m1 = 1 << 20
    threads = os.cpu_count() or 1
    memcpy_gbs = O.lib().oracle_memcpy_bw(64 << 20, threads, 5) / 1e9
    for nm in ("ag_bidir_ring8", "ag_ring8_2_4_7"):
        js = load_schedule(nm)
        d = json.loads(js)
        p2 = sccl.LoopbackPlan(js, m1, sccl.U8, device=0)
        us = graph_time_us(p2, [x[:m1] for x in send], [x[:P * m1] for x in recv], stream, 50)
        p2.close()
        ins = O.seeded_inputs("allgather", P, m1, O.U8, 0)
        ex = O.Execution(d, ins, m1, O.U8, check=True)
        row = {"gpu_us": round(us, 2)}
        for th in (1, threads):
            ex.run(th)
            ts = []
            for _ in range(20):
                t0 = time.perf_counter()
                ex.run(th)
                ts.append(time.perf_counter() - t0)
            row[f"cpu_{th}t_us_median"] = round(1e6 * statistics.median(ts), 1)
            row[f"cpu_{th}t_us_min"] = round(1e6 * min(ts), 1)
        # host bytes the CPU executor moves: every receipt read + written, plus the local slots
        host_bytes = 2 * (len(d["sends"]) * m1 // (d["G"] // P))
        row["cpu_host_bytes"] = host_bytes
        row["cpu_memcpy_roofline_us"] = round(host_bytes / (memcpy_gbs * 1e9) * 1e6, 1)
        c1[f"{nm} ({d['C']},{d['S']},{d['R']})"] = row
    c1["host_memcpy_GBps"] = round(memcpy_gbs, 1)
    c1["host_threads"] = threads
    c1["host_cpu"] = host_cpu()
    out["config1_cpu_vs_gpu_1MiB"] = c1

    # the same lowered program as per-op cudaMemcpyAsync copies (the paper's
    # per-step copy lowering): a library-copy executor's speed
    if plan.info()["protocol"] != "ll":
        for r in recv:
            r.zero_()
        torch.cuda.synchronize()
        plan.launch_copy_engine(send, recv, stream)
        stream.synchronize()
        want = torch.cat(send)
        assert all(torch.equal(r, want) for r in recv), "bench: copy-engine result wrong"
        ca, cb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ca.record(stream)
        for _ in range(3):
            plan.launch_copy_engine(send, recv, stream)
        cb.record(stream)
        stream.synchronize()
        ce_ms = ca.elapsed_time(cb) / 3
        m = send[0].numel()
        out["copy_engine_baseline"] = {
            "ms": round(ce_ms, 3), "busbw_per_rank_GBps": round(busbytes("allgather", P, m) / (ce_ms * 1e-3) / 1e9, 2),
            "note": "same lowered program, one cudaMemcpyAsync D2D per op output, step order, one stream"}
        plan.launch(send, recv, stream)  # leave the plan's buffers in the kernel's state
        stream.synchronize()
    return out


def allreduce_e2e(sccl, xs, ys, stream):
    """BASELINE config 3 end to end: allreduce (8,2,2) bf16 at 64 MiB per
    rank through the public API with host buffers (H2D every rank's input,
    D2H every rank's output, per step), with the CPU reference executor on a
    bounded sample beside it."""
    import torch
    P, M = len(xs), xs[0].numel()
    nm = "ar_oneshot_full8"
    plan = sccl.LoopbackPlan(load_schedule(nm), M, sccl.BF16, device=0)
    hin = [torch.randint(-16, 17, (M // 2,), dtype=torch.int16).to(torch.bfloat16).view(torch.uint8).pin_memory()
           for _ in range(P)]
    hout = torch.empty(P * M, dtype=torch.uint8, pin_memory=True)
    steps = 5
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        for i in range(steps + 1):
            if i == 1:
                a.record(stream)
            for h, x in zip(hin, xs):
                x.copy_(h, non_blocking=True)
            plan.launch(xs, ys, stream)
            for r in range(P):
                hout[r * M:(r + 1) * M].copy_(ys[r], non_blocking=True)
        b.record(stream)
    stream.synchronize()
    plan.check()
    plan.close()
    ms = a.elapsed_time(b) / steps
    want = torch.stack([h.view(torch.bfloat16).double() for h in hin]).sum(0).to(torch.bfloat16).view(torch.uint8)
    assert all(torch.equal(hout[r * M:(r + 1) * M], want) for r in range(P)), "allreduce e2e wrong"
    # CPU reference on a bounded sample (4 MiB per rank, 1 thread and all threads)
    O = _oracle()
    d = json.loads(load_schedule(nm))
    ms_cpu = {}
    for th in (1, os.cpu_count() or 1):
        ins = O.seeded_inputs("allreduce", P, 4 << 20, O.BF16, 0)
        ex = O.Execution(d, ins, 4 << 20, O.BF16, check=True)
        ex.run(th)
        t0 = time.perf_counter()
        for _ in range(5):
            ex.run(th)
        ms_cpu[th] = (time.perf_counter() - t0) / 5 * 1e3
    bb = busbytes("allreduce", P, M)
    return {"workload": "allreduce (8,2,2) bf16, 64 MiB per rank, 8 loopback ranks",
            "e2e": {"value": round(bb / (ms * 1e-3) / 1e9, 3), "unit": "GB/s", "h2d_bytes_per_step": P * M,
                    "d2h_bytes_per_step": P * M, "ms_per_step": round(ms, 3)},
            "cpu_baseline": [{"value": round(busbytes("allreduce", P, 4 << 20) / (t * 1e-3) / 1e9, 3), "unit": "GB/s",
                              "cores": th, "kind": "port",
                              "sample": "oracle executor, ar_oneshot_full8, 8 ranks x 4 MiB bf16, per-rank bus GB/s"}
                             for th, t in ms_cpu.items()]}


# --------------------------------------------------------------------------- CPU reference (bounded)
def cpu_reference_run(P: int, js: str, m: int, seconds: float, threads: int):
    """Time the oracle executor loop on the same schedule; returns
    (aggregate bus GB/s over the P ranks, seconds, runs)."""
    O = _oracle()
    d = json.loads(js)
    ins = O.seeded_inputs(d["collective"], P, m, O.U8, 0)
    ex = O.Execution(d, ins, m, O.U8, check=True)
    ex.run(threads)  # warm-up
    n, t0 = 0, time.perf_counter()
    while True:
        ex.run(threads)
        n += 1
        dt = time.perf_counter() - t0
        if dt >= seconds:
            break
    return P * busbytes("allgather", P, m) * n / dt / 1e9, dt, n


# --------------------------------------------------------------------------- GPU, N > 1
def nvlink_counters(index: int):
    """NVML NVLink 5 byte counters of GPU `index`, summed over its links:
    (tx bytes, rx bytes, field source) or None.  Fields 202 / 204
    (NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES / _RCV_BYTES) per link; fallback
    138 / 139 (THROUGHPUT_DATA_TX / RX, KiB)."""
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(index)
        for tx_id, rx_id, scale in ((202, 204, 1), (138, 139, 1024)):
            try:
                reqs = [(tx_id, l) for l in range(18)] + [(rx_id, l) for l in range(18)]
                vals = pynvml.nvmlDeviceGetFieldValues(h, reqs)
                tx = rx = 0
                ok = 0
                for req, v in zip(reqs, vals):
                    if v.nvmlReturn != 0:
                        continue
                    ok += 1
                    x = int(v.value.ullVal) * scale
                    if req[0] == tx_id:
                        tx += x
                    else:
                        rx += x
                if ok:
                    return tx, rx, f"NVML field {tx_id}/{rx_id} over {ok // 2} links"
            except Exception:
                continue
    except Exception:
        return None
    return None


def tune_nchannels(dist, sccl, js, rank, P, nbytes, dtype, dev_index, args, send, stream, tdev):
    """CTAs per rank of a one-rank-per-GPU plan: the multi-process policy
    table's default (fitted on a loopback proxy) against
    16 and 64, 5 launches each into the plan's registered buffer, max over
    ranks.  Returns (nchannels to use, {nchannels: (request, ms)})."""
    import torch
    tune = {}
    for cand in (0, 16, 64):
        tp = sccl.Plan(js, rank, P, nbytes, dtype, device=dev_index, nchannels=cand, tile_bytes=args.tile,
                       mem_handles=args.mem, timeout_ms=BENCH_TIMEOUT_MS)
        try:
            tp.bind_with()
            treg, _ = tp.recv_buffer()
            for _ in range(2):
                tp.launch(send, treg, stream)
            dist.barrier()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(5):
                tp.launch(send, treg, stream)
            b.record()
            torch.cuda.synchronize()
            tp.check()
            t = torch.tensor([a.elapsed_time(b) / 5], device=tdev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            tune[tp.info()["nchannels"] if cand == 0 else cand] = (cand, round(float(t), 4))
        finally:
            tp.close()
    return min(tune.values(), key=lambda x: x[1])[0], tune


def run_multi(args):
    import torch
    import torch.distributed as dist
    from paper_2008_08708_b200 import sccl
    t_start = time.perf_counter()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    # SCCL_BENCH_SHARE_GPU=1: every rank on cuda:0 (validates this path on a
    # one-GPU box; the ranks time-slice one GPU, so its numbers are not
    # performance).  NCCL refuses duplicate GPUs: gloo, no NCCL baselines.
    shared = os.environ.get("SCCL_BENCH_SHARE_GPU") == "1"
    mps = shared and bool(os.environ.get("CUDA_MPS_PIPE_DIRECTORY"))  # ranks concurrent under MPS, not time-sliced
    dev_index = 0 if shared else local
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    if shared:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=dev)
    P = world
    name = workload_schedule(P, args.schedule)
    js = load_schedule(name)
    m = args.bytes
    g = torch.Generator(device=dev)
    g.manual_seed(1000 + rank)
    send = torch.randint(0, 256, (m,), dtype=torch.uint8, device=dev, generator=g)
    recv = torch.empty(P * m, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()
    # CTAs per rank: the multi-process policy table's default (32) was fitted
    # on a loopback proxy, so on a real NVLink box the
    # bench first times the default against 16 and 64 (max over ranks, a few
    # launches each) and runs the workload with the fastest; the line reports
    # every candidate.  --nchannels N pins it.
    tune = {}
    nch_use = args.nchannels
    # (not in shared-GPU mode: there every rank's CTAs share one GPU's slots,
    # and a 64-CTA candidate x P ranks need not be co-resident under MPS)
    if args.nchannels == 0 and not shared:
        nch_use, tune = tune_nchannels(dist, sccl, js, rank, P, m, sccl.U8, dev_index, args, send, stream,
                                       "cpu" if shared else dev)
    plan = sccl.Plan(js, rank, P, m, sccl.U8, device=dev_index, nchannels=nch_use, tile_bytes=args.tile,
                     mem_handles=args.mem, timeout_ms=BENCH_TIMEOUT_MS)
    plan.bind_with()
    for _ in range(args.warmup):
        plan.launch(send, recv, stream)
    torch.cuda.synchronize()
    ref = gather_ref(dist, send, P, shared, dev)
    # recorded, not asserted: a rank that raised here would leave its peers
    # waiting in the next collective; the line reports every rank's result
    same = [None] * P
    dist.all_gather_object(same, bool(torch.equal(ref, recv)))
    regptr, _ = plan.recv_buffer()
    oracle_ok = multi_oracle_check(dist, sccl, rank, P, dev_index, args.mem)

    def timed(fn, steps):
        dist.barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(steps):
            fn()
        b.record()
        torch.cuda.synchronize()
        t = torch.tensor([a.elapsed_time(b) / steps], device="cpu" if shared else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)  # max over ranks
        return float(t)

    n0 = plan.launch_count
    nv0 = nvlink_counters(dev_index)
    with ClockSampler(dev_index) as clk:
        ms = timed(lambda: plan.launch(send, regptr, stream), args.steps)
    nv1 = nvlink_counters(dev_index)
    launches = plan.launch_count - n0
    plan.check()
    per_rank = busbytes("allgather", P, m) / (ms * 1e-3) / 1e9
    traffic = None
    traffic_src = None
    if nv0 and nv1 and not shared:
        traffic = (nv1[0] - nv0[0]) / args.steps  # TX bytes per launch of this GPU
        traffic_src = f"{nv1[2]}, TX bytes per launch around the timed region (rank {rank})"
    traffic_all = [None] * P
    dist.all_gather_object(traffic_all, traffic)

    # e2e through the public API with pinned host buffers: this rank's input
    # H2D, the collective, this rank's whole output D2H, every step
    hs = torch.empty(m, dtype=torch.uint8, pin_memory=True)
    hs.copy_(send.cpu())
    hr = torch.empty(P * m, dtype=torch.uint8, pin_memory=True)

    def e2e_step():
        send.copy_(hs, non_blocking=True)
        plan.launch(send, recv, stream)
        hr.copy_(recv, non_blocking=True)
    e2e_ms = timed(e2e_step, max(3, min(args.steps, 10)))
    baselines = {} if (shared or args.no_sweep) else nccl_baselines(args, dist, sccl, rank, P, dev, dev_index,
                                                                     send, ref, ms, timed, t_start)
    if rank == 0:
        line = {
            "metric": METRIC, "value": round(per_rank * P, 2), "unit": "GB/s", "n_gpus": 1 if shared else P,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic (uniform random bytes)",
            "config": {"workload": (f"{sched_label(name)}; {P} ranks as {P} processes "
                                    + ("running concurrently on ONE GPU under MPS (the multi-process kernel path "
                                       "timed with every rank in one HBM: no NVLink)" if mps else
                                       "time-sliced on ONE GPU (multi-process path validation, not performance)"))
                       if shared
                       else _workload_text(P, P, name, multi=True),
                       "ranks": P, "bytes_per_rank": m, "schedule_file": f"tests/golden/schedules/bench/{name}.json",
                       "parallelism": f"ranks{P}", "nchannels": plan.info()["nchannels"],
                       "nchannels_autotune_ms": {str(k): v[1] for k, v in tune.items()} or None,
                       "l2": "no flush: buffers >> L2", "shared_gpu": shared, "mem_handles": args.mem,
                       "value_convention": "sum over GPUs of per-rank bus GB/s (nccl-tests busBW)"},
            "busbw_per_rank_GBps": round(per_rank, 2),
            "oracle_check": {"bytes_per_rank": 65536, "ranks_bit_exact": oracle_ok},
            "workload_check": {"what": "every rank's output of the timed workload == torch.distributed all_gather "
                                       "of the inputs", "ranks_equal": same},
            "roofline": {"bound": "nvlink", "achieved": round(per_rank, 1), "peak": NVLINK_PEAK, "unit": "GB/s",
                         "frac": round(per_rank / NVLINK_PEAK, 4), "traffic": traffic_all[0],
                         "traffic_per_rank": traffic_all, "traffic_source": traffic_src,
                         "algorithmic_bytes_per_launch": busbytes("allgather", P, m),
                         "peak_source": "nominal NVLink 5 per direction per GPU"},
            "e2e": {"value": round(busbytes("allgather", P, m) * P / (e2e_ms * 1e-3) / 1e9, 3), "unit": "GB/s",
                    "h2d_bytes_per_step": P * m, "d2h_bytes_per_step": P * P * m,
                    "note": "every rank: H2D of its input + collective + D2H of its whole output, per step; "
                            "sum over GPUs"},
            "clocks": clk.summary(), "gpu_launches": launches,
        }
        line.update(baselines)
        print(json.dumps(line), flush=True)
    plan.close()
    dist.destroy_process_group()


def gather_ref(dist, send, P, shared, dev):
    import torch
    m = send.numel()
    if shared:
        parts = [torch.empty(m, dtype=torch.uint8) for _ in range(P)]
        dist.all_gather(parts, send.cpu())
        return torch.cat(parts).to(dev)
    ref = torch.empty(P * m, dtype=torch.uint8, device=dev)
    dist.all_gather_into_tensor(ref, send)
    torch.cuda.synchronize()
    return ref


def multi_oracle_check(dist, sccl, rank, P, dev_index, mem):
    """Every rank's output of the workload schedule at 64 KiB per rank against
    the CPU oracle's (digest); returns the per-rank results (rank 0)."""
    import torch
    O = _oracle()
    name = workload_schedule(P, "auto")
    js = load_schedule(name)
    d = json.loads(js)
    nb = 65536
    ins = O.seeded_inputs(d["collective"], P, nb, O.U8, 9)
    want = O.execute(d, ins, nb, O.U8)[rank]
    plan = sccl.Plan(js, rank, P, nb, sccl.U8, device=dev_index, mem_handles=mem, timeout_ms=BENCH_TIMEOUT_MS)
    plan.bind_with()
    recv = torch.zeros(want.size, dtype=torch.uint8, device=f"cuda:{dev_index}")
    plan.launch(torch.from_numpy(ins[rank]).to(recv.device), recv)
    torch.cuda.synchronize()
    plan.check()
    ok = O.digest([recv.cpu().numpy()]) == O.digest([want])
    plan.close()
    res = [None] * P
    dist.all_gather_object(res, ok)
    return res


def nccl_baselines(args, dist, sccl, rank, P, dev, dev_index, send, ref, ms_ours, timed, t_start):
    """Same-box NCCL (NCCL_PROTO=Simple; alltoall
    as grouped send/recv) beside the executor, each timed
    the same way (max over ranks).  Every NCCL configuration gets its own
    communicator, created while its NCCL_* variables are set.

    Each comparison is a section: value checks are recorded (never asserted),
    an exception is caught and reported under the section's key after every
    rank has agreed on the outcome, and a section starts only while the run is
    younger than EXTRAS_BUDGET_S (rank 0 decides for all) -- so one failed or
    slow comparison costs its own key, not the bench line."""
    import torch
    m = send.numel()
    out = {}

    def section(key, fn):
        go = [time.perf_counter() - t_start < EXTRAS_BUDGET_S]
        dist.broadcast_object_list(go, src=0)
        if not go[0]:
            out[key] = {"skipped": f"bench extras budget ({EXTRAS_BUDGET_S:.0f} s) spent"}
            return
        err = None
        try:
            res = fn()
        except Exception as e:  # noqa: BLE001 -- reported in the line
            res, err = None, f"{type(e).__name__}: {e}"[:400]
        errs = [None] * P
        dist.all_gather_object(errs, err)
        if any(errs):
            out[key] = {"error": {r: e for r, e in enumerate(errs) if e}}
        else:
            out[key] = res

    def group_with(env):
        old = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        try:
            grp = dist.new_group(backend="nccl")
            t = torch.zeros(1, device=dev)
            dist.all_reduce(t, group=grp)  # the communicator is created now, with env in force
            torch.cuda.synchronize()
        finally:
            for k, v in old.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v
        return grp

    g_simple = group_with({"NCCL_PROTO": "Simple"})
    g_ring = group_with({"NCCL_ALGO": "Ring"})
    g_tree = group_with({"NCCL_ALGO": "Tree"})
    g_ll = group_with({"NCCL_PROTO": "LL"})  # SURVEY.md 8(d) cfg 3: NCCL_PROTO=Simple/LL/LL128
    g_ll128 = group_with({"NCCL_PROTO": "LL128"})
    bw = lambda coll, nbytes, t: round(busbytes(coll, P, nbytes) / (t * 1e-3) / 1e9, 2)

    def agree(ok):
        """every rank's check result (collective)"""
        res = [None] * P
        dist.all_gather_object(res, bool(ok))
        return res

    def allgather():  # at the workload size
        ag = {"ours_ms": round(ms_ours, 4), "ours_busbw": bw("allgather", m, ms_ours)}
        for tag, grp in (("nccl_default", None), ("nccl_simple", g_simple)):
            t = timed(lambda: dist.all_gather_into_tensor(ref, send, group=grp), args.steps)
            ag[f"{tag}_ms"], ag[f"{tag}_busbw"] = round(t, 4), bw("allgather", m, t)
        return ag
    section("nccl_allgather", allgather)

    # allreduce bf16 at 64 MiB: our one-shot (and Hamiltonian at P=2/8) vs NCCL Ring / Tree / default
    M = 64 << 20
    x = torch.randint(-16, 17, (M // 2,), device=dev).to(torch.bfloat16)
    y = torch.empty_like(x)
    z_ref = x.clone()
    dist.all_reduce(z_ref)
    torch.cuda.synchronize()

    def allreduce():
        ar = {"bytes_per_rank": M}
        for nm in ([f"ar_oneshot_full{P}"] + ([f"ar_ham_full{P}"] if P in (2, 8) else [])):
            nch, tn = tune_nchannels(dist, sccl, load_schedule(nm), rank, P, M, sccl.BF16, dev_index, args,
                                     x.view(torch.uint8), torch.cuda.current_stream(), dev)
            ar[f"ours_{nm}_nchannels_autotune_ms"] = {str(k): v[1] for k, v in tn.items()}
            p2 = sccl.Plan(load_schedule(nm), rank, P, M, sccl.BF16, device=dev_index, mem_handles=args.mem,
                           timeout_ms=BENCH_TIMEOUT_MS, nchannels=nch)
            try:
                p2.bind_with()
                reg, _ = p2.recv_buffer()
                p2.launch(x.view(torch.uint8), reg)
                t = timed(lambda: p2.launch(x.view(torch.uint8), reg), args.steps)
                p2.launch(x.view(torch.uint8), y.view(torch.uint8))
                torch.cuda.synchronize()
                p2.check()
                ar[f"ours_{nm}_ms"], ar[f"ours_{nm}_busbw"] = round(t, 4), bw("allreduce", M, t)
                # integer-valued bf16 inputs: the sum is exact in any order
                ar[f"ours_{nm}_equals_nccl"] = agree(torch.equal(y, z_ref))
            finally:
                p2.close()
        for tag, grp in (("nccl_default", None), ("nccl_ring", g_ring), ("nccl_tree", g_tree),
                         ("nccl_simple", g_simple), ("nccl_ll", g_ll), ("nccl_ll128", g_ll128)):
            z = x.clone()
            t = timed(lambda: dist.all_reduce(z, group=grp), args.steps)
            ar[f"{tag}_ms"], ar[f"{tag}_busbw"] = round(t, 4), bw("allreduce", M, t)
        return ar
    section("nccl_allreduce_bf16", allreduce)

    # the switch-offloaded comparison backend, only when
    # every rank's device can join a multicast team
    sup = [None] * P
    dist.all_gather_object(sup, bool(sccl.nvls_supported(dev_index, P)))

    def nvls():
        if not all(sup):
            return {"skipped": f"no multicast team (nvls_supported per rank: {sup})"}
        nv = sccl.NvlsAllreduce(rank, P, M, sccl.BF16, device=dev_index, timeout_ms=BENCH_TIMEOUT_MS)
        try:
            nv.launch(x, y)
            torch.cuda.synchronize()
            nv.check()
            r = {"bytes_per_rank": M, "equals_nccl": agree(torch.equal(y, z_ref))}
            t = timed(lambda: nv.launch(), args.steps)  # in its multicast-bound buffer (zero-copy)
            nv.check()
            r["ours_nvls_ms"], r["ours_nvls_busbw"] = round(t, 4), bw("allreduce", M, t)
            return r
        finally:
            nv.close()
    section("nvls_allreduce_bf16", nvls)

    def alltoall():  # at 64 MiB: direct (P,1,1) vs NCCL grouped send/recv
        a_in = torch.randint(0, 256, (M,), dtype=torch.uint8, device=dev)
        a_out = torch.empty_like(a_in)
        nch, tune_a2a = tune_nchannels(dist, sccl, load_schedule(f"a2a_direct_full{P}"), rank, P, M, sccl.U8,
                                       dev_index, args, a_in, torch.cuda.current_stream(), dev)
        p3 = sccl.Plan(load_schedule(f"a2a_direct_full{P}"), rank, P, M, sccl.U8, device=dev_index,
                       mem_handles=args.mem, timeout_ms=BENCH_TIMEOUT_MS, nchannels=nch)
        try:
            p3.bind_with()
            reg3, _ = p3.recv_buffer()
            t = timed(lambda: p3.launch(a_in, reg3), args.steps)
            p3.launch(a_in, a_out)
            chk = torch.empty_like(a_in)
            dist.all_to_all_single(chk, a_in)
            torch.cuda.synchronize()
            p3.check()
            same = agree(torch.equal(chk, a_out))
            tn = timed(lambda: dist.all_to_all_single(chk, a_in), args.steps)
            return {"bytes_per_rank": M, "ours_nchannels_autotune_ms": {str(k): v[1] for k, v in tune_a2a.items()},
                    "ours_ms": round(t, 4), "ours_busbw": bw("alltoall", M, t),
                    "nccl_ms": round(tn, 4), "nccl_busbw": bw("alltoall", M, tn), "equals_nccl": same}
        finally:
            p3.close()
    section("nccl_alltoall", alltoall)

    # latency sweep (<= 64 KB) and bandwidth points (>= 64 MB): allgather with
    # the cost model's per-size choice among this P's schedule files
    def sweep():
        cands = [n for n in (f"ag_oneshot_full{P}", f"ag_ring_ring{P}", f"ag_ham_full{P}")
                 if os.path.exists(os.path.join(SCHED_DIR, n + ".json"))]
        texts = [load_schedule(n) for n in cands]
        pts = []
        sizes = (1 << 10, 4 << 10, 16 << 10, 64 << 10, 1 << 20, 64 << 20, 256 << 20)
        s_all = torch.randint(0, 256, (max(sizes),), dtype=torch.uint8, device=dev)  # (not the workload's m bytes)
        r_all = torch.empty(P * max(sizes), dtype=torch.uint8, device=dev)
        for sz in sizes:
            i, proto, _ = sccl.select(texts, sz, sccl.U8, multiprocess=True)
            p4 = sccl.Plan(texts[i], rank, P, sz, sccl.U8, device=dev_index, protocol=proto, mem_handles=args.mem,
                           timeout_ms=BENCH_TIMEOUT_MS)
            try:
                p4.bind_with()
                reg4, _ = p4.recv_buffer()
                s4 = s_all[:sz]
                r4 = r_all[:P * sz]
                iters = 200 if sz <= (64 << 10) else 20
                t = timed(lambda: p4.launch(s4, reg4), iters)
                p4.check()
                tn = timed(lambda: dist.all_gather_into_tensor(r4, s4), iters)
                tns = timed(lambda: dist.all_gather_into_tensor(r4, s4, group=g_simple), iters)
                pts.append({"bytes_per_rank": sz, "schedule": cands[i], "protocol": proto,
                            "ours_us": round(t * 1e3, 2), "nccl_us": round(tn * 1e3, 2),
                            "nccl_simple_us": round(tns * 1e3, 2), "ours_busbw": bw("allgather", sz, t),
                            "nccl_busbw": bw("allgather", sz, tn)})
            finally:
                p4.close()
        return pts
    section("allgather_sweep_vs_nccl", sweep)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--bytes", type=int, default=128 << 20, help="per-rank allgather input")
    ap.add_argument("--schedule", default="auto", choices=["auto", "ham", "oneshot", "ring"])
    ap.add_argument("--nchannels", type=int, default=0)
    ap.add_argument("--mem", default="ipc", choices=["ipc", "vmm"],
                    help="N>1: share plan regions through CUDA IPC handles or VMM (cuMem) fds")
    ap.add_argument("--tile", type=int, default=0)
    ap.add_argument("--ref-bytes", type=int, default=0,
                    help="--impl reference: bytes per rank (0 = the GPU arm's --bytes)")
    ap.add_argument("--cpu-bytes", type=int, default=16 << 20)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-sweep", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    elif (args.gpus == 1 and "WORLD_SIZE" not in os.environ or os.environ.get("WORLD_SIZE") == "1") and \
            os.environ.get("SCCL_BENCH_FORCE_MULTI") != "1":
        run_loopback(args)
    else:
        if "RANK" not in os.environ:
            sys.exit(f"bench.py --gpus {args.gpus}: launch one process per GPU with torchrun, e.g. python -m "
                     f"torch.distributed.run --nnodes=1 --nproc-per-node {args.gpus} --master-addr 127.0.0.1 "
                     f"bench.py --gpus {args.gpus}")
        run_multi(args)


if __name__ == "__main__":
    main()
