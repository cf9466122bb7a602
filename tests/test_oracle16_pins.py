"""Pins of the packed-half oracle (P:L98 __half2, SPEC S1: round
after every add/min/FMA).  CPU only.  The references here share nothing with the C code:

* round_half against numpy's float32 -> float16 conversion (correctly rounded, RNE) on
  random values and against every finite binary16 value (round trip, SPEC invariant);
* the cell against exact rational arithmetic + an independent Python RNE-to-binary16;
* brute force over all warp paths at <= 5 x 9 with that independent cell (the min-then-add
  DP equals the min over path folds because rounding is monotone);
* closed form N = 1 and the exact embedding (a half-exact cut scores 0).
"""
from fractions import Fraction

import numpy as np
import pytest

HALF_MAX = Fraction(65504)


def _rne_half(v: Fraction) -> Fraction:
    """Round an exact rational to binary16 (RNE, subnormals, overflow -> inf as None)."""
    if v == 0:
        return Fraction(0)
    sgn = -1 if v < 0 else 1
    a = abs(v)
    e = 0
    while a >= 2 ** (e + 1):
        e += 1
    while a < 2 ** e:
        e -= 1
    ulp = Fraction(2) ** (e - 10) if e >= -14 else Fraction(2) ** -24
    q = a / ulp
    fl = q.numerator // q.denominator
    frac = q - fl
    if frac > Fraction(1, 2) or (frac == Fraction(1, 2) and fl % 2 == 1):
        fl += 1
    r = fl * ulp
    if r > HALF_MAX:
        return None
    return sgn * r


def _cell16(x, y, m):
    t = _rne_half(Fraction(float(x)) - Fraction(float(y)))
    return _rne_half(t * t + Fraction(float(m)))


def test_round_half_matches_numpy_random(oracle_mod):
    rng = np.random.default_rng(16)
    vals = np.concatenate([rng.standard_normal(4000) * 10.0, rng.standard_normal(2000) * 1e-5,
                           rng.uniform(60000, 70000, 500)]).astype(np.float32)
    for v in vals:
        assert np.float32(oracle_mod.round_half(float(v))) == np.float32(np.float16(v)), v


def test_round_half_roundtrip_every_finite_half(oracle_mod):
    h = np.arange(0, 0x7C00, dtype=np.uint16).view(np.float16)   # +0 .. 65504
    for x in h[::7].astype(np.float32):                           # every 7th pattern (9,070 values)
        assert oracle_mod.round_half(float(x)) == float(x)
        assert oracle_mod.round_half(-float(x)) == -float(x)


def test_cell16_matches_exact_rational(oracle_mod):
    """Two rows, one column: cost = cell(x1, y, cell(x0, y, 0)) -- the C cell with a non-zero
    addend against exact rationals + the independent RNE (including overflow to +inf)."""
    rng = np.random.default_rng(17)
    for k in range(400):
        scale = 10.0 ** rng.integers(-3, 3)
        x = (rng.standard_normal(2) * scale).astype(np.float16).astype(np.float32)
        y = np.float32(np.float16(rng.standard_normal() * scale))
        if k % 50 == 0:
            x[0], y = np.float32(200.0), np.float32(-60.0)        # forces overflow to +inf
        d0 = _cell16(x[0], y, 0)
        want = None if d0 is None else _cell16(x[1], y, d0)
        r = oracle_mod.sdtw(x[:, None].reshape(1, 2), np.array([y], np.float32), half=True)
        got = float(r["cost"][0])
        if want is None:
            assert got == float("inf")
        else:
            assert Fraction(got) == want, (x, y)


def _brute16(x, Y):
    N, M = len(x), len(Y)
    best = None
    best_end = None
    for s in range(M):
        stack = [(0, s, _cell16(x[0], Y[s], 0))]
        while stack:
            i, j, v = stack.pop()
            if v is None:
                continue
            if i == N - 1 and (best is None or v < best or (v == best and j < best_end)):
                best, best_end = v, j
            for di, dj in ((1, 1), (1, 0), (0, 1)):
                a, b = i + di, j + dj
                if a < N and b < M:
                    stack.append((a, b, _cell16(x[a], Y[b], v)))
    return best, best_end


@pytest.mark.parametrize("inst", range(12))
def test_half_dp_equals_brute_force(oracle_mod, inst):
    rng = np.random.default_rng(1600 + inst)
    N, M = int(rng.integers(1, 5)), int(rng.integers(1, 9))
    x = (rng.standard_normal(N) * (3 if inst % 2 else 0.01)).astype(np.float16).astype(np.float32)
    Y = (rng.standard_normal(M) * (3 if inst % 2 else 0.01)).astype(np.float16).astype(np.float32)
    bc, be = _brute16(x, Y)
    r = oracle_mod.sdtw(x[None], Y, half=True)
    assert Fraction(float(r["cost"][0])) == bc and r["end"][0] == be


def test_half_closed_form_single_row(oracle_mod):
    rng = np.random.default_rng(18)
    x = np.float32(np.float16(rng.standard_normal()))
    Y = rng.standard_normal(200).astype(np.float16).astype(np.float32)
    vals = [_cell16(x, y, 0) for y in Y]
    best = min(vals)
    r = oracle_mod.sdtw(np.array([[x]], np.float32), Y, half=True, start=True)
    assert Fraction(float(r["cost"][0])) == best and r["end"][0] == vals.index(best) == r["start"][0]


def test_half_embedding_scores_zero(oracle_mod):
    rng = np.random.default_rng(19)
    Y = rng.standard_normal(3000).astype(np.float32)
    s, L = 777, 200
    r = oracle_mod.sdtw(Y[s:s + L][None], Y, half=True, start=True)
    assert r["cost"][0] == 0 and r["end"][0] == s + L - 1 and r["start"][0] == s


def test_half_differs_from_fp32_within_paper_tolerance(oracle_mod):
    """fp16 accumulation: relative error vs the fp32 DP ~1e-2 (SURVEY NEXT-1 tolerance)."""
    from datagen import nanopore_queries, nanopore_reference
    Y = oracle_mod.znorm(nanopore_reference(20_000, 2)[None])[0]
    Q = oracle_mod.znorm(nanopore_queries(8, 500, 20_000, 2))
    a = oracle_mod.sdtw(Q, Y)["cost"]
    b = oracle_mod.sdtw(Q, Y, half=True)["cost"]
    rel = np.abs(a.astype(np.float64) - b) / np.maximum(a, 1e-3)
    assert np.all(rel < 3e-2), rel
