#!/usr/bin/env python3
"""Write the canonical schedule files bench.py runs (tests/golden/schedules/
bench/*.json).  Both arms read these files: the GPU executor through the
C-ABI and `bench.py --impl reference` through the CPU oracle, which must not
import the product package.  tests/test_bench_schedules.py checks the files
against this generator."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2008_08708_b200 import sccl  # noqa: E402
from paper_2008_08708_b200 import schedules as S  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "schedules", "bench")


def bench_schedules():
    """name -> canonical schedule JSON"""
    out = {}
    # P = 1 (a local copy): bench.py's multi-process path self-test on one GPU
    # (SCCL_BENCH_FORCE_MULTI=1 with one torchrun rank: a real NCCL communicator)
    one1 = S.one_shot_allgather(1)
    out["ag_oneshot_full1"] = sccl.canonicalize(S.to_json(one1))
    out["ar_oneshot_full1"] = sccl.canonicalize(S.allreduce_from(one1))
    out["a2a_direct_full1"] = sccl.canonicalize(S.to_json(S.direct_alltoall(1)))
    for P in (2, 4, 8):
        one = S.one_shot_allgather(P)
        out[f"ag_oneshot_full{P}"] = sccl.canonicalize(S.to_json(one))
        out[f"ag_ring_ring{P}"] = sccl.canonicalize(S.to_json(S.ring_allgather(P)))
        out[f"ar_oneshot_full{P}"] = sccl.canonicalize(S.allreduce_from(one))
        out[f"ar_ring_ring{P}"] = sccl.canonicalize(S.allreduce_from(S.ring_allgather(P)))
        out[f"a2a_direct_full{P}"] = sccl.canonicalize(S.to_json(S.direct_alltoall(P)))
        if P not in (4, 6):  # K_4* has no Hamiltonian decomposition
            ham = S.hamiltonian_allgather(P)
            out[f"ag_ham_full{P}"] = sccl.canonicalize(S.to_json(ham))
            out[f"ar_ham_full{P}"] = sccl.canonicalize(S.allreduce_from(ham))
    # BASELINE config 1: the ring(8) latency-optimal allgathers (1,4,4), (2,4,7)
    out["ag_bidir_ring8"] = sccl.canonicalize(S.to_json(S.bidir_ring_allgather(8)))
    with open(os.path.join(ROOT, "tests", "golden", "schedules", "ag_ring8_2_4_7.json")) as f:
        out["ag_ring8_2_4_7"] = sccl.canonicalize(f.read())
    return out


def main():
    os.makedirs(OUT, exist_ok=True)
    for name, js in bench_schedules().items():
        with open(os.path.join(OUT, name + ".json"), "w") as f:
            f.write(js + "\n")
    print(f"wrote {len(bench_schedules())} schedules to {OUT}")


if __name__ == "__main__":
    main()
