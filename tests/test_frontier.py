"""Topology discovery -> synthesis target -> candidates -> per-size choice
(SURVEY.md 8(f) f2 -> f1 -> f3)."""
import json
import os
import socket
import subprocess
import sys

import pytest

from paper_2008_08708_b200 import frontier, sccl

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_index_lists_switch_frontiers():
    """The NVSwitch synthesis target has committed frontiers at P = 2/4/8
    (per-GPU egress / ingress groups): bandwidth-optimal R/C =
    P - 1 under that model."""
    idx = frontier.index()
    for P in (2, 4, 8):
        sw = [e for e in idx if e["topology"] == f"switch:{P}"]
        assert sw, P
        assert any(e["bandwidth_optimal"] and e["R"] == (P - 1) * e["C"] for e in sw)
    for e in idx:
        with open(os.path.join(frontier.FRONTIER_DIR, e["file"])) as f:
            d = json.loads(f.read())
        assert (d["C"], d["S"], d["R"]) == (e["C"], e["S"], e["R"]) and d["topology"]["name"] == e["topology"]


def test_targets_and_candidates():
    assert frontier.targets_for("switch:8") == ["switch:8", "full:8"]
    assert frontier.targets_for("loopback:1", 8) == ["switch:8", "full:8", "ring:8"]
    ag = frontier.candidates("allgather", "switch:8", 8)
    assert len(ag) >= 2 and all(sccl.verify(js) == [] for js in ag)
    ar = frontier.candidates("allreduce", "switch:8", 8)
    assert len(ar) == len(ag)
    for js in ar:
        d = json.loads(js)
        assert d["collective"] == "allreduce" and sccl.verify(js) == []
    with pytest.raises(ValueError):
        frontier.candidates("allgather", "dgx1")


def test_choice_per_size_changes_with_size():
    """Latency-optimal entry at small sizes, a bandwidth-optimal one at large
    sizes (the cost model's switch between implementations)."""
    cands = frontier.candidates("allgather", "loopback:1", 8)
    small = frontier.choose(cands, 1024)
    large = frontier.choose(cands, 256 << 20)
    d_small = json.loads(cands[small[0]])
    assert small[1] == "ll" and large[1] == "simple"
    assert d_small["S"] <= min(json.loads(c)["S"] for c in cands) + 1


def test_machine_discovery_on_cpu_raises():
    """No GPU: discovery finds no target (no silent default)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        frontier.for_this_machine("allgather", 8)


WORKER = r"""
import sys
sys.path.insert(0, {root!r})
import torch.distributed as dist
from paper_2008_08708_b200 import frontier, sccl
rank = int(sys.argv[1])
dist.init_process_group("gloo", init_method="tcp://127.0.0.1:{port}", rank=rank, world_size=2)
ap = sccl.AutoPlan(frontier.candidates("allreduce", "switch:2", 2), rank, 2, sccl.BF16, device=-1)
out = []
for nb in (1024, 1 << 20, 64 << 20):
    i, proto, plan = ap.plan_for(nb)
    out.append((i, proto, plan.info()["program"]["fingerprint"]))
print("CHOICES", out, flush=True)
ap.close()
dist.destroy_process_group()
"""


def test_autoplan_binds_per_size_across_ranks(tmp_path):
    """Multi-process AutoPlan (gloo, world 2, host-only plans): every rank
    makes the same per-size choice, lowers the same program and binds."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    script = tmp_path / "w.py"
    script.write_text(WORKER.format(root=ROOT, port=port))
    procs = [subprocess.Popen([sys.executable, str(script), str(r)], stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                              text=True) for r in range(2)]
    outs = [p.communicate(timeout=120) for p in procs]
    for p, (o, e) in zip(procs, outs):
        assert p.returncode == 0, e[-2000:]
    lines = [o.split("CHOICES", 1)[1].strip() for o, _ in outs]
    assert lines[0] == lines[1]
