"""bench.py's driver contract on CPU: the reference arm prints one JSON line
with the contract's keys (single process, and rank 0 only under a 2-rank
launch), and the GPU arm fails loudly -- no CPU fallback -- where there is
no GPU."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BENCH = os.path.join(ROOT, "bench.py")
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"}


def _lines(out):
    return [json.loads(x) for x in out.splitlines() if x.startswith("{")]


def test_reference_arm_line():
    r = subprocess.run([sys.executable, BENCH, "--impl", "reference", "--bytes", "65536", "--steps", "3",
                        "--warmup", "3"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _lines(r.stdout)
    assert len(lines) == 1
    d = lines[0]
    assert KEYS <= set(d), KEYS - set(d)
    assert d["impl"] == "reference" and d["higher_is_better"] is True and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["e2e"]["value"] == d["value"] and d["cpu_baseline"]["value"] == d["value"]
    assert d["cpu_baseline"]["kind"] in ("port", "reference") and d["cpu_baseline"]["cores"] >= 1
    assert d["config"]["same_config"] is True and d["config"]["bytes_per_rank"] == 65536
    assert d["config"]["ranks"] == 8 and d["warmup"] >= 3


def test_reference_arm_under_two_ranks_prints_on_rank0_only():
    outs = []
    for rank in (0, 1):
        env = dict(os.environ, RANK=str(rank), LOCAL_RANK=str(rank), WORLD_SIZE="2", MASTER_ADDR="127.0.0.1")
        r = subprocess.run([sys.executable, BENCH, "--impl", "reference", "--gpus", "2", "--bytes", "65536",
                            "--steps", "3", "--warmup", "3"], capture_output=True, text=True, timeout=300, cwd=ROOT,
                           env=env)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(_lines(r.stdout))
    assert len(outs[0]) == 1 and outs[1] == []
    d = outs[0][0]
    assert d["n_gpus"] == 2 and d["config"]["ranks"] == 2 and d["impl"] == "reference"


def _has_gpu():
    import torch
    return torch.cuda.is_available()


@pytest.mark.skipif(_has_gpu(), reason="a GPU is present")
def test_gpu_arm_fails_loudly_without_a_gpu():
    r = subprocess.run([sys.executable, BENCH, "--steps", "3", "--warmup", "3", "--bytes", "65536"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode != 0
    assert _lines(r.stdout) == []
