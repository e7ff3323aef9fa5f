"""(alpha, beta) cost model and per-size algorithm selection.

Restates the reference's costmodel module:
a k-synchronous schedule (C, S, R) moving L bytes costs S*alpha + (R/C)*L*beta
(exact rational arithmetic), two schedules cross at
L* = (S_b - S_a) * alpha / ((R_a/C_a - R_b/C_b) * beta), and
best_for_size picks the cheapest frontier entry per size, ties to fewer steps
(SPEC.md:485-493).

On B200 the model is calibrated from the executor's own measured latency
sweep (``fit``), and ``select`` chooses among lowered candidate schedules for
a buffer size -- the runtime "switch between multiple implementations
based on the input size" of PAPER.md:1037.
"""
from __future__ import annotations

from fractions import Fraction
from typing import Dict, Iterable, List, NamedTuple, Optional, Sequence, Tuple


class Algo(NamedTuple):
    """A k-synchronous schedule's cost coordinates in the reference's order
    (time(S, R, C, ...), crossover(a: (S,R,C), b: (S,R,C)))."""
    S: int
    R: int
    C: int


Tuple3 = Tuple[int, int, int]  # (S, R, C), as in the reference


def _algo(x) -> Algo:
    """(S, R, C) tuple or Algo; a mapping with S/R/C keys also works."""
    if isinstance(x, dict):
        return Algo(int(x["S"]), int(x["R"]), int(x["C"]))
    S, R, C = x
    return Algo(int(S), int(R), int(C))


def _q(x) -> Fraction:
    return x if isinstance(x, Fraction) else Fraction(x)


def time(S: int, R: int, C: int, alpha, beta, L) -> Fraction:
    """S*alpha + (R/C)*L*beta, exact."""
    if C == 0:
        raise ValueError("C must be >= 1")
    return S * _q(alpha) + Fraction(R, C) * _q(L) * _q(beta)


def crossover(a: Tuple3, b: Tuple3, alpha, beta) -> Optional[Fraction]:
    """Size where time_a == time_b, or None for parallel / dominated lines
    (SPEC.md:476-484).  a, b are (S, R, C), the reference's order."""
    Sa, Ra, Ca = _algo(a)
    Sb, Rb, Cb = _algo(b)
    slope = (Fraction(Ra, Ca) - Fraction(Rb, Cb)) * _q(beta)
    icpt = (Sb - Sa) * _q(alpha)
    if slope == 0:
        return None
    L = icpt / slope
    return L if L > 0 else None


def best_for_size(frontier: Sequence[Tuple3], alpha, beta, sizes: Iterable) -> List[Tuple[object, Tuple3]]:
    """Per size, the entry minimizing time; ties -> fewer steps
    (SPEC.md:485-493).  Entries are (S, R, C); each is returned as given."""
    if not frontier:
        raise ValueError("empty frontier")
    out = []
    for L in sizes:
        best = min(frontier, key=lambda e: (time(*_algo(e), alpha, beta, L), _algo(e).S))
        out.append((L, best))
    return out


def fit(points: Sequence[Tuple[int, int, int, float, float]]) -> Tuple[float, float]:
    """Least-squares (alpha, beta) from measurements (S, R, C, bytes, seconds)."""
    import numpy as np
    A = np.array([[S, R / C * L] for S, R, C, L, _ in points], dtype=float)
    y = np.array([t for *_, t in points], dtype=float)
    sol, *_ = np.linalg.lstsq(A, y, rcond=None)
    return float(max(sol[0], 0.0)), float(max(sol[1], 0.0))


def select(candidates: Dict[str, Tuple3], alpha: float, beta: float, nbytes: int) -> str:
    """Name of the candidate schedule (S, R, C) the model predicts fastest
    for nbytes (per-rank buffer; L = nbytes)."""
    a = Fraction(alpha).limit_denominator(10**12)
    b = Fraction(beta).limit_denominator(10**18)
    return min(candidates, key=lambda k: (time(*_algo(candidates[k]), a, b, nbytes), _algo(candidates[k]).S))
