"""Statistics helpers of the reference library (include/escg/stats.hpp, src/stats.cpp) restated as TEST
INFRASTRUCTURE (SURVEY §2.1 marks stats.cpp out of scope for the product): the statistical parity tests
use them as checkers.  Nothing in paper_2508_16639_b200/ imports this module.

    mean_std(xs)                     stats.cpp:9-21   sample mean and (n-1) standard deviation
    gamma_q(a, x)                    stats.cpp:61-66  regularized upper incomplete gamma Q(a, x)
    chi_square_uniform_pvalue(bins)  stats.cpp:68-81  P(chi2 >= observed) for equiprobable bins
    ks_two_sample_pvalue(a, b)       stats.cpp:83-110 asymptotic two-sample Kolmogorov-Smirnov p

Invalid arguments raise ValueError (the reference's std::invalid_argument).
"""
from __future__ import annotations

import math
from typing import Sequence

from dataclasses import dataclass


@dataclass
class MeanStd:
    mean: float = 0.0
    std_dev: float = 0.0
    n: int = 0


def mean_std(xs: Sequence[float]) -> MeanStd:
    """stats.cpp:9-21: sample mean and (n-1) standard deviation (0 when n < 2)."""
    r = MeanStd(n=len(xs))
    if not xs:
        return r
    r.mean = sum(xs) / len(xs)
    if len(xs) >= 2:
        r.std_dev = math.sqrt(sum((x - r.mean) ** 2 for x in xs) / (len(xs) - 1))
    return r

_EPS = 1e-15
_TINY = 1e-300


def _log_prefactor(a: float, x: float) -> float:
    return -x + a * math.log(x) - math.lgamma(a)


def _gamma_p_series(a: float, x: float) -> float:
    """P(a, x) = x^a e^-x / Gamma(a) * sum_k x^k / (a (a+1) ... (a+k)); for x < a + 1."""
    term = 1.0 / a
    total = term
    denom = a
    for _ in range(500):
        denom += 1.0
        term *= x / denom
        total += term
        if abs(term) < abs(total) * _EPS:
            break
    return total * math.exp(_log_prefactor(a, x))


def _gamma_q_continued_fraction(a: float, x: float) -> float:
    """Q(a, x) by the modified Lentz evaluation of its continued fraction; for x >= a + 1."""
    b = x + 1.0 - a
    c = 1.0 / _TINY
    d = 1.0 / b
    h = d
    for i in range(1, 500):
        an = -i * (i - a)
        b += 2.0
        d = an * d + b
        if abs(d) < _TINY:
            d = _TINY
        c = b + an / c
        if abs(c) < _TINY:
            c = _TINY
        d = 1.0 / d
        delta = d * c
        h *= delta
        if abs(delta - 1.0) < _EPS:
            break
    return h * math.exp(_log_prefactor(a, x))


def gamma_q(a: float, x: float) -> float:
    if a <= 0.0 or x < 0.0:
        raise ValueError("gamma_q requires a > 0 and x >= 0")
    if x == 0.0:
        return 1.0
    if x < a + 1.0:
        return 1.0 - _gamma_p_series(a, x)
    return _gamma_q_continued_fraction(a, x)


def chi_square_uniform_pvalue(bin_counts: Sequence[int]) -> float:
    counts = [int(c) for c in bin_counts]
    if len(counts) < 2:
        raise ValueError("need at least two bins")
    total = sum(counts)
    if total == 0:
        raise ValueError("need at least one sample")
    expected = total / len(counts)
    chi2 = sum((c - expected) ** 2 / expected for c in counts)
    return gamma_q((len(counts) - 1) / 2.0, chi2 / 2.0)


def ks_two_sample_pvalue(a: Sequence[float], b: Sequence[float]) -> float:
    if len(a) == 0 or len(b) == 0:
        raise ValueError("KS test needs non-empty samples")
    xa, xb = sorted(float(v) for v in a), sorted(float(v) for v in b)
    na, nb = len(xa), len(xb)
    # sup |F_a - F_b| over the pooled sample points (ties advance both empirical CDFs together)
    d, i, j = 0.0, 0, 0
    while i < na and j < nb:
        x = min(xa[i], xb[j])
        while i < na and xa[i] <= x:
            i += 1
        while j < nb and xb[j] <= x:
            j += 1
        d = max(d, abs(i / na - j / nb))
    ne = na * nb / (na + nb)
    lam = (math.sqrt(ne) + 0.12 + 0.11 / math.sqrt(ne)) * d
    # Kolmogorov survival function Q_KS(lambda) = 2 sum_k (-1)^(k-1) exp(-2 k^2 lambda^2)
    p, sign = 0.0, 1.0
    for k in range(1, 101):
        term = math.exp(-2.0 * k * k * lam * lam)
        p += 2.0 * sign * term
        sign = -sign
        if term < 1e-12:
            break
    return min(1.0, max(0.0, p))


def correlation_length(cells, length: int, height: int, rmax: int = 64) -> float:
    """Spatial correlation length of one lattice (test-side observable, not a reference function):
    C(r) = P(s(x) = s(x + r)) - sum_s rho_s^2 over horizontal and vertical periodic displacements r,
    l = the first r with C(r) <= C(0)/e, linearly interpolated (rmax if never).  The same estimator
    is applied to device and reference lattices, so only its distribution is compared."""
    import numpy as np

    a = np.asarray(cells).reshape(height, length)
    rmax = min(rmax, min(length, height) // 4)
    rho = np.bincount(a.ravel().astype(np.int64)) / a.size
    base = float((rho ** 2).sum())
    prev = None
    c0 = None
    for r in range(rmax + 1):
        same = 0.5 * ((a == np.roll(a, r, axis=1)).mean() + (a == np.roll(a, r, axis=0)).mean())
        c = same - base
        if r == 0:
            c0 = c
            prev = c
            continue
        thr = c0 / math.e
        if c <= thr:
            return (r - 1) + (prev - thr) / (prev - c) if prev != c else float(r)
        prev = c
    return float(rmax)


def bootstrap_threshold(grid, outcomes, n_boot: int = 2000, seed: int = 0):
    """Mobility threshold = first M (ascending) with P(coexist) < 1/2, and its bootstrap distribution
    (trials resampled with replacement per M).  outcomes[i] = 0/1 coexistence per trial at grid[i].
    Returns (threshold or None, list of bootstrap thresholds, None where no M falls below 1/2)."""
    import numpy as np

    rng = np.random.default_rng(seed)
    grid = list(grid)

    def thr(ps):
        for m, p in zip(grid, ps):
            if p < 0.5:
                return m
        return None

    point = thr([float(np.mean(o)) for o in outcomes])
    boots = []
    for _ in range(n_boot):
        boots.append(thr([float(np.mean(rng.choice(o, size=len(o), replace=True))) for o in outcomes]))
    return point, boots
