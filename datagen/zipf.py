"""Bounded Zipf sampling (input generation only).

The paper's skew observation: "20% of IDs will cover 70% by average and up to 99%" of the
training data (Fig. investigation).  We model a field's ID popularity as
a bounded Zipf law p(r) = r^-alpha / H(V, alpha), r = 1..V (SPEC.md L40-48 uses the same
family), and sample it exactly with Hoermann & Derflinger's rejection-inversion method
(ACM TOMACS 6(3), 1996), vectorised in numpy.
"""
from __future__ import annotations

import numpy as np


def _helper1(x):  # log1p(x)/x, stable near 0
    out = np.ones_like(x)
    nz = np.abs(x) > 1e-8
    out[nz] = np.log1p(x[nz]) / x[nz]
    out[~nz] = 1.0 - x[~nz] * (0.5 - x[~nz] / 3.0)
    return out


def _helper2(x):  # expm1(x)/x, stable near 0
    out = np.ones_like(x)
    nz = np.abs(x) > 1e-8
    out[nz] = np.expm1(x[nz]) / x[nz]
    out[~nz] = 1.0 + x[~nz] * 0.5 * (1.0 + x[~nz] / 3.0)
    return out


class ZipfSampler:
    """Exact sampler of p(r) ∝ r^-alpha on r in [1, V] (alpha >= 0)."""

    def __init__(self, V: int, alpha: float):
        assert V >= 1 and alpha >= 0
        self.V, self.a = int(V), float(alpha)
        self.hx1 = self._H(np.array([1.5]))[0] - 1.0
        self.hN = self._H(np.array([self.V + 0.5]))[0]
        self.s = 2.0 - self._Hinv(np.array([self._H(np.array([2.5]))[0] - self._h(np.array([2.0]))[0]]))[0]

    def _h(self, x):
        return np.exp(-self.a * np.log(x))

    def _H(self, x):
        lx = np.log(x)
        return _helper2((1.0 - self.a) * lx) * lx

    def _Hinv(self, x):
        t = x * (1.0 - self.a)
        t = np.maximum(t, -1.0)
        return np.exp(_helper1(t) * x)

    def sample(self, rng: np.random.Generator, n: int) -> np.ndarray:
        """n ranks in [1, V] (int64)."""
        out = np.empty(n, np.int64)
        todo = np.arange(n)
        if self.V == 1:
            out[:] = 1
            return out
        while todo.size:
            u = self.hN + rng.random(todo.size) * (self.hx1 - self.hN)
            x = self._Hinv(u)
            k = np.floor(x + 0.5)
            k = np.clip(k, 1, self.V)
            acc = (k - x <= self.s) | (u >= self._H(k + 0.5) - self._h(k))
            out[todo[acc]] = k[acc].astype(np.int64)
            todo = todo[~acc]
        return out


def zipf_head_mass(V: int, alpha: float, head_fraction: float) -> float:
    """Closed form: share of draws that fall in the top ceil(head_fraction*V) ranks."""
    k = int(np.ceil(head_fraction * V))
    r = np.arange(1, V + 1, dtype=np.float64)
    w = r ** (-alpha)
    return float(w[:k].sum() / w.sum())


def resolve_alpha(V: int, head_fraction: float = 0.2, head_mass: float = 0.7) -> float:
    """Bisection for alpha such that the head covers head_mass."""
    lo, hi = 0.0, 4.0
    for _ in range(60):
        mid = 0.5 * (lo + hi)
        if zipf_head_mass(V, mid, head_fraction) < head_mass:
            lo = mid
        else:
            hi = mid
    return 0.5 * (lo + hi)
