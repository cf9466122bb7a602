"""Exact fp32 helpers for the oracle pins (tests only).

fma_f32 computes the correctly rounded fp32 value of a*b+c from exact rational
arithmetic -- an FMA that shares nothing with libm's fmaf (which the oracle
uses), so the closed-form pins are independent of the oracle's arithmetic.
"""
from fractions import Fraction

import numpy as np


def round_f32(v: Fraction) -> np.float32:
    """Round an exact rational to the nearest fp32 (ties to even)."""
    c = np.float32(float(v))
    best = c
    bd = abs(Fraction(float(c)) - v) if np.isfinite(c) else None
    if bd is None:
        return c
    for nb in (np.nextafter(c, np.float32(-np.inf)), np.nextafter(c, np.float32(np.inf))):
        if not np.isfinite(nb):
            continue
        d = abs(Fraction(float(nb)) - v)
        if d < bd or (d == bd and (int(np.float32(nb).view(np.uint32)) & 1) == 0):
            best, bd = nb, d
    return np.float32(best)


def fma_f32(a, b, c) -> np.float32:
    return round_f32(Fraction(float(np.float32(a))) * Fraction(float(np.float32(b)))
                     + Fraction(float(np.float32(c))))


def cell_f32(x, y, m, fma: bool) -> np.float32:
    """d(x,y)+m for one cell: t = fl(x-y), then fma(t,t,m) or fl(fl(t*t)+m)."""
    t = np.float32(np.float32(x) - np.float32(y))
    if fma:
        return fma_f32(t, t, m)
    return np.float32(np.float32(t * t) + np.float32(m))


def fold_f32(xs, y, fma: bool) -> np.float32:
    """Left fold c_0 = cell(x_0, y, 0), c_i = cell(x_i, y, c_{i-1})."""
    c = np.float32(0.0)
    for x in xs:
        c = cell_f32(x, y, c, fma)
    return c


def dp_f64(x, Y):
    """fp64 sDTW by the plain definition (tests: accuracy bound, small sizes)."""
    x = np.asarray(x, np.float64)
    Y = np.asarray(Y, np.float64)
    N, M = x.shape[0], Y.shape[0]
    prev = np.zeros(M)           # virtual row -1
    for i in range(N):
        cur = np.empty(M)
        d = (x[i] - Y) ** 2
        diag_prev = 0.0 if i == 0 else np.inf
        left = np.inf
        for j in range(M):
            m = min(diag_prev, prev[j], left)
            cur[j] = d[j] + m
            diag_prev = prev[j]
            left = cur[j]
        prev = cur
    return float(prev.min()), int(prev.argmin()), prev
