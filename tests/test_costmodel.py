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
    rng = random.Random(0)
    for _ in range(5):
        a = F(rng.randint(1, 10**6), rng.randint(1, 1000))
        b = F(rng.randint(1, 10**6), rng.randint(1, 10**9))
        assert cm.crossover((2, 2, 3), (6, 3, 7), a, b) == 3 * a / b
    assert cm.crossover((1, 2, 2), (1, 2, 2), 1, 1) is None
    assert cm.crossover((1, 2, 2), (2, 2, 2), 1, 1) is None  # same S: one dominates


def test_best_for_size_flips_at_crossover():
    a, b = F(5), F(1, 100)
    fr = [(2, 2, 3), (6, 3, 7)]
    Ls = cm.crossover(fr[0], fr[1], a, b)
    res = dict(cm.best_for_size(fr, a, b, [Ls / 2, Ls * 2]))
    assert res[Ls / 2] == (2, 2, 3) and res[Ls * 2] == (6, 3, 7)
    small, large = cm.best_for_size([(1, 2, 2), (6, 3, 7)], a, b, [0, 10**12])
    assert small[1] == (1, 2, 2) and large[1] == (6, 3, 7)


def test_fit_and_select():
    alpha, beta = 3e-6, 1 / 500e9
    pts = []
    for (C, S, R) in ((1, 1, 1), (7, 7, 7), (1, 7, 7)):
        for L in (1 << 10, 1 << 16, 1 << 20, 1 << 24):
            pts.append((C, S, R, L, S * alpha + R / C * L * beta))
    fa, fb = cm.fit(pts)
    assert abs(fa - alpha) / alpha < 1e-6 and abs(fb - beta) / beta < 1e-6
    cands = {"oneshot": (1, 1, 1), "777": (7, 7, 7), "ring": (1, 7, 7)}
    assert cm.select(cands, fa, fb, 1024) == "oneshot"


def test_topology_discovery_degrades_on_cpu():
    from paper_2008_08708_b200 import topology
    info = topology.discover()
    assert "target" in info
    import torch
    if not torch.cuda.is_available():
        assert info["target"] == "unknown"
