"""The schedule files bench.py reads (both arms) are the canonical
serializations of the generators (tools/make_bench_schedules.py) and verify."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
from make_bench_schedules import OUT, bench_schedules  # noqa: E402

from paper_2008_08708_b200 import sccl  # noqa: E402

SCHED = bench_schedules()


@pytest.mark.parametrize("name", sorted(SCHED))
def test_bench_schedule_file_matches_generator(name):
    with open(os.path.join(OUT, name + ".json")) as f:
        text = f.read().strip()
    assert text == SCHED[name]
    assert sccl.verify(text) == []
