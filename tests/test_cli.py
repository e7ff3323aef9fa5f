"""The C++ CLI (the reference's cmd_verify / cmd_exec)."""
import json
import os
import subprocess

import numpy as np
import pytest

import oracle as O
from paper_2008_08708_b200 import sccl

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2008_08708_b200", "lib", "sccl-exec")
SCHED = os.path.join(ROOT, "tests", "golden", "schedules")


def test_verify_exit_codes(tmp_path):
    ok = subprocess.run([CLI, "verify", os.path.join(SCHED, "ag_ring8_2_4_7.json")], capture_output=True, text=True)
    assert ok.returncode == 0 and ok.stdout.strip() == "Ok"
    d = json.load(open(os.path.join(SCHED, "ag_ring8_2_4_7.json")))
    d["sends"] = d["sends"][:-1]
    bad = tmp_path / "bad.json"
    bad.write_text(json.dumps(d))
    r = subprocess.run([CLI, "verify", str(bad)], capture_output=True, text=True)
    assert r.returncode == 1 and "post" in r.stdout + r.stderr or "violation" in r.stdout
    r = subprocess.run([CLI, "frobnicate", str(bad)], capture_output=True, text=True)
    assert r.returncode == 1


def test_cli_payload_rule():
    a = O.cli_payload(20, 3, 1)
    assert a.size == 20 and O.fnv1a(a) != O.fnv1a(O.cli_payload(20, 3, 2))


@pytest.mark.gpu
@pytest.mark.parametrize("name,dtype", [("ag_ring8_2_4_7", "u8"), ("ar_from_dgx1_2_2_3", "i32"),
                                        ("a2a_dgx1_8_2_3", "u8"), ("ar_from_ring8_2_4_7", "bf16")])
def test_exec_digest_matches_oracle(name, dtype):
    path = os.path.join(SCHED, name + ".json")
    nbytes = 8 * 4096
    out = subprocess.run([CLI, "exec", path, "--bytes", str(nbytes), "--seed", "7", "--dtype", dtype],
                         capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    res = json.loads(out.stdout)
    d = json.load(open(path))
    sb, _ = O.buffer_sizes(d["collective"], d["P"], nbytes)
    ins = [O.cli_payload(sb, 7, r) for r in range(d["P"])]
    ref = O.execute(d, ins, nbytes, O.DTYPE_NAMES[dtype])
    assert res["digests"] == [O.fnv1a(r) for r in ref]


@pytest.mark.gpu
@pytest.mark.parametrize("name,dtype,protocol", [("ag_ring8_2_4_7", "u8", "auto"), ("ar_from_dgx1_2_2_3", "i32", "simple"),
                                                 ("a2a_dgx1_8_2_3", "u8", "ll"), ("ar_from_ring8_2_4_7", "bf16", "ll")])
def test_exec_mp_digest_matches_oracle(name, dtype, protocol):
    """`sccl-exec exec-mp`: the C++-host use of the multi-process boundary --
    one forked process per rank, plan create / export / file-based handle
    exchange / bind / two launches through the C-ABI only -- gives the
    oracle's digests on every rank (all ranks on cuda:0 here, time-sliced)."""
    path = os.path.join(SCHED, name + ".json")
    nbytes = 8 * 4096
    out = subprocess.run([CLI, "exec-mp", path, "--bytes", str(nbytes), "--seed", "9", "--dtype", dtype,
                          "--protocol", protocol], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    res = json.loads(out.stdout)
    d = json.load(open(path))
    assert res["processes"] == d["P"]
    sb, _ = O.buffer_sizes(d["collective"], d["P"], nbytes)
    ins = [O.cli_payload(sb, 9, r) for r in range(d["P"])]
    ref = O.execute(d, ins, nbytes, O.DTYPE_NAMES[dtype])
    assert res["digests"] == [O.fnv1a(r) for r in ref]
