"""Cost model, acceptance criterion 8."""
import random
from fractions import Fraction as F

from paper_2008_08708_b200 import costmodel as cm


def test_time_examples():
    a, b, L = F(3), F(1, 7), F(1000)
    assert cm.time(7, 7, 6, a, b, L) == 7 * a + F(7, 6) * L * b  # PAPER §2.4
    assert cm.time(5, 9, 2, a, b, 0) == 5 * a
    assert cm.time(2, 3, 2, a, b, L) == 2 * a + F(3, 2) * L * b


def test_crossover_3alpha_over_beta():
    """(2,3,2) vs (3,7,6) -> L* = 3 alpha / beta, tuples in the
    reference's (S, R, C) order."""
    rng = random.Random(0)
    for _ in range(5):
        a = F(rng.randint(1, 10**6), rng.randint(1, 1000))
        b = F(rng.randint(1, 10**6), rng.randint(1, 10**9))
        assert cm.crossover((2, 3, 2), (3, 7, 6), a, b) == 3 * a / b
        assert cm.crossover(cm.Algo(S=2, R=3, C=2), cm.Algo(S=3, R=7, C=6), a, b) == 3 * a / b
    assert cm.crossover((2, 3, 2), (2, 3, 2), 1, 1) is None  # identical tuples
    assert cm.crossover((2, 3, 2), (2, 7, 6), 1, 1) is None  # same S: one dominates


def test_best_for_size_flips_at_crossover():
    """SPEC.md:488-492, (S, R, C) tuples."""
    a, b = F(5), F(1, 100)
    fr = [(2, 3, 2), (3, 7, 6)]
    Ls = cm.crossover(fr[0], fr[1], a, b)
    res = dict(cm.best_for_size(fr, a, b, [Ls / 2, Ls * 2]))
    assert res[Ls / 2] == (2, 3, 2) and res[Ls * 2] == (3, 7, 6)
    small, large = cm.best_for_size([(2, 2, 1), (3, 7, 6)], a, b, [0, 10**12])
    assert small[1] == (2, 2, 1) and large[1] == (3, 7, 6)


def test_fit_and_select():
    alpha, beta = 3e-6, 1 / 500e9
    pts = []
    for (S, R, C) in ((1, 1, 1), (7, 7, 7), (7, 7, 1)):
        for L in (1 << 10, 1 << 16, 1 << 20, 1 << 24):
            pts.append((S, R, C, L, S * alpha + R / C * L * beta))
    fa, fb = cm.fit(pts)
    assert abs(fa - alpha) / alpha < 1e-6 and abs(fb - beta) / beta < 1e-6
    cands = {"oneshot": (1, 1, 1), "777": (7, 7, 7), "ring": (7, 7, 1)}
    assert cm.select(cands, fa, fb, 1024) == "oneshot"


def test_topology_discovery_degrades_on_cpu():
    from paper_2008_08708_b200 import topology
    info = topology.discover()
    assert "target" in info
    import torch
    if not torch.cuda.is_available():
        assert info["target"] == "unknown"
