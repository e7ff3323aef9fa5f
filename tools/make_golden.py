#!/usr/bin/env python3
"""Generate tests/golden/*.json: the known-answer schedules and vectors that
pin the oracle (the reference ships no executable; these restate its
textual examples).

Each fixture holds the canonical schedule text, the payload recipe (seeded
PRNG or explicit values), and the expected per-rank output digests.  The
digests are produced by the C oracle and must agree with the independent
pure-Python restatement before they are written.  Explicit-value KATs also
carry the literal expected bytes from the SPEC text.

Usage: python tools/make_golden.py   (rewrites tests/golden/)
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]

import numpy as np  # noqa: E402

import oracle as O  # noqa: E402
from paper_2008_08708_b200 import schedules as S  # noqa: E402
from paper_2008_08708_b200 import sccl  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def vec_case(name, js, nbytes, dtype, seed, mode, source, extra=None):
    d = json.loads(js)
    ins = O.seeded_inputs(d["collective"], d["P"], nbytes, dtype, seed, mode)
    a = O.execute(d, ins, nbytes, dtype)
    b = O.execute_py(d, ins, nbytes, dtype)
    assert all(np.array_equal(x, y) for x, y in zip(a, b)), name
    fx = {"name": name, "source": source, "schedule": js, "bytes_per_rank": nbytes,
          "dtype": dtype, "seed": seed, "mode": mode,
          "input_digest": O.digest(ins), "output_digests": [O.digest([x]) for x in a]}
    if extra:
        fx.update(extra)
    return fx


def main():
    os.makedirs(OUT, exist_ok=True)
    fixtures = []

    # 2-node send of payload 0xAB -> node 1 slot holds 0xAB
    fixtures.append({"name": "kat_two_node_send", "source": "SPEC.md:424",
                     "schedule": S.to_json(S.two_node_send()), "bytes_per_rank": 1, "dtype": O.U8,
                     "inputs_hex": ["ab", "00"], "expected_hex": ["ab", "ab"]})
    # 2-node Reduce with values 3 and 4 -> root holds 7
    red = S.reduce_from(S.two_node_send())
    fixtures.append({"name": "kat_two_node_reduce", "source": "SPEC.md:425",
                     "schedule": red, "bytes_per_rank": 4, "dtype": O.I32,
                     "inputs_hex": [np.int32(3).tobytes().hex(), np.int32(4).tobytes().hex()],
                     "expected_hex": [np.int32(7).tobytes().hex(), None]})

    # SPEC.md:406-408 verifier KATs on the Fig. 2 schedule
    fig2 = json.loads(S.to_json(S.recursive_doubling_ring4()))
    deleted = dict(fig2, sends=fig2["sends"][1:])
    shifted = dict(fig2, sends=[[c, a, b, 0] for c, a, b, _ in fig2["sends"]], rounds=[1, 2])
    fixtures.append({"name": "kat_verify_fig2", "source": "SPEC.md:406-408",
                     "schedule": json.dumps(fig2), "expect": "ok",
                     "mutants": [{"schedule": json.dumps(deleted), "expect_kind": "post"},
                                 {"schedule": json.dumps(shifted), "expect_kind": "bandwidth"}]})
    # SPEC.md:415-417 combining verifier KATs
    rs_fig2 = sccl.invert(S.recursive_doubling_ring4())
    dup = json.loads(rs_fig2)
    dup["sends"] = dup["sends"] + [dup["sends"][0][:3] + [dup["sends"][0][3]]]
    fixtures.append({"name": "kat_verify_combining", "source": "SPEC.md:415-417",
                     "schedule": red, "expect": "ok",
                     "mutants": [{"schedule": json.dumps(dup), "expect_kind": "multiplicity"}],
                     "also_ok": [rs_fig2]})

    # executor vectors (seeded), oracle C == oracle Python
    ag_dgx = S.dgx1_allgather_122()
    fixtures.append(vec_case("ar_dgx1_8_4_4_int", S.allreduce_from(ag_dgx), 4096, O.I32, 641, "random",
                             "SPEC.md:426, acceptance SPEC.md:641 (the (8,4,4) Table 4 row); exact sums",
                             {"check_direct_sum": True}))
    # the SPEC's own (48,6,14) row: RS+AG of the SMT-synthesized DGX-1 (6,3,7)
    with open(os.path.join(OUT, "schedules", "ar_from_dgx1_6_3_7.json")) as f:
        ar48 = f.read().strip()
    fixtures.append(vec_case("ar_dgx1_48_6_14_int", ar48, 6144, O.I32, 641, "random",
                             "SPEC.md:426, acceptance SPEC.md:641: DGX-1 Allreduce (48,6,14), random integer "
                             "payloads, all 8 nodes hold the direct sum", {"check_direct_sum": True}))
    fixtures.append(vec_case("ag_fig2_u8", S.to_json(S.recursive_doubling_ring4()), 1000, O.U8, 1, "random",
                             "Fig. 2 (PAPER.md:309-312)"))
    fixtures.append(vec_case("ag_777_u8", S.to_json(S.hamiltonian_allgather(8)), 4096 + 48, O.U8, 2, "random",
                             "BASELINE config 2 (C,S,R)=(7,7,7) on full(8)"))
    fixtures.append(vec_case("ag_ring8_144_u8", S.to_json(S.bidir_ring_allgather(8)), 1 << 14, O.U8, 3, "random",
                             "BASELINE config 1 (1,4,4) on ring(8) (Table 5, PAPER.md:952)"))
    fixtures.append(vec_case("a2a_881_u8", S.to_json(S.direct_alltoall(8)), 8 * 520, O.U8, 4, "random",
                             "BASELINE config 4 (8,1,1) on full(8)"))
    ar777 = S.allreduce_from(S.hamiltonian_allgather(8))
    for dt, nm in ((O.F32, "f32"), (O.BF16, "bf16"), (O.F16, "f16"), (O.I32, "i32")):
        fixtures.append(vec_case(f"ar_56_14_14_{nm}", ar777, 8192, dt, 5, "random",
                                 "BASELINE config 3, fixed reduction order (DESIGN.md)"))
    fixtures.append(vec_case("ar_822_bf16_smallint", S.allreduce_from(S.one_shot_allgather(8)), 8192, O.BF16, 6,
                             "smallint", "BASELINE config 3 (8,2,2); order-independent exact sums",
                             {"check_direct_sum": True}))
    fixtures.append(vec_case("rs_ring8_f32", S.reducescatter_from(S.ring_allgather(8)), 4096, O.F32, 7, "random",
                             "inverted ring allgather (SPEC.md:338-346)"))
    fixtures.append(vec_case("reduce_chain_bf16", S.reduce_from(S.pipelined_chain_broadcast(5, 4, 2)), 4096,
                             O.BF16, 8, "random", "inverted chain broadcast (SPEC.md:338)"))

    for f in os.listdir(OUT):
        if f.endswith(".json"):
            os.remove(os.path.join(OUT, f))
    for fx in fixtures:
        with open(os.path.join(OUT, fx["name"] + ".json"), "w") as f:
            json.dump(fx, f, indent=1, sort_keys=True)
            f.write("\n")
    print(f"wrote {len(fixtures)} fixtures to {OUT}")


if __name__ == "__main__":
    main()
