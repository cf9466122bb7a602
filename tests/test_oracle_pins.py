"""Pins of the CPU oracle against things other than itself.

Every test here runs without a GPU.  Each pin is chosen so that a plausible
mistake in oracle/sdtw_oracle.c (dropped neighbour, wrong boundary, swapped
roles of query/reference, wrong tie rule, wrong variance) fails at least one:

* printed worked examples (tests/golden/*.json, SPEC.md S:L261/L270/L271/L190/L199)
* brute-force enumeration of all warp paths (tests/pins/brute.c) -- bit exact
* closed forms: N=1, M=1, constant reference (exact rational FMA in tests/_exact.py)
* invariants: embedding, time stretch, reference prefix / extension, reversal
* start validity by a DP restricted to one start column; walk-back == forward
* fp64 definition within the fp32 error bound
* normaliser fixtures, fp64 re-check, affine invariance
"""
import ctypes
import json
import os

import numpy as np
import pytest

from tests._exact import cell_f32, dp_f64, fold_f32

GOLD = os.path.join(os.path.dirname(__file__), "golden")
f32p = ctypes.POINTER(ctypes.c_float)
i64p = ctypes.POINTER(ctypes.c_int64)


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def _brute(L, x, Y, fma):
    x = np.ascontiguousarray(x, np.float32)
    Y = np.ascontiguousarray(Y, np.float32)
    row = np.empty(Y.shape[0], np.float32)
    c = ctypes.c_float()
    e = ctypes.c_int64()
    L.brute_sdtw(x.ctypes.data_as(f32p), x.shape[0], Y.ctypes.data_as(f32p), Y.shape[0], int(fma),
                 row.ctypes.data_as(f32p), ctypes.byref(c), ctypes.byref(e))
    return np.float32(c.value), e.value, row


def _restricted(L, x, Y, fma, s, end):
    x = np.ascontiguousarray(x, np.float32)
    Y = np.ascontiguousarray(Y, np.float32)
    a = np.empty(Y.shape[0], np.float32)
    b = np.empty(Y.shape[0], np.float32)
    return np.float32(L.restricted_dp(x.ctypes.data_as(f32p), x.shape[0], Y.ctypes.data_as(f32p),
                                      Y.shape[0], int(fma), int(s), int(end),
                                      a.ctypes.data_as(f32p), b.ctypes.data_as(f32p)))


@pytest.mark.parametrize("fma", [True, False])
@pytest.mark.parametrize("name", ["spec_worked_example_1.json", "spec_worked_example_2.json",
                                  "tie_example_zeros.json"])
def test_golden_fixtures(oracle_mod, name, fma):
    g = _gold(name)
    x = np.array(g["query"], np.float32)
    Y = np.array(g["reference"], np.float32)
    D, S = oracle_mod.sdtw_full(x, Y, fma=fma)
    assert np.array_equal(D, np.array(g["matrix"], np.float32))
    r = oracle_mod.sdtw(x, Y, fma=fma, start=True)
    assert r["cost"][0] == np.float32(g["cost"])
    assert r["end"][0] == g["end"]
    assert r["start"][0] == g["start"]
    assert oracle_mod.walkback(D, g["end"]) == g["start"]


@pytest.mark.parametrize("fma", [True, False])
def test_brute_force_6x12(oracle_mod, brute_lib, fma):
    """BASELINE.json config 1: brute-force path enumeration at 6x12, bit exact."""
    for inst in range(150):
        rng = np.random.default_rng(1001 + inst)
        N = int(rng.integers(1, 7))
        M = int(rng.integers(1, 13))
        if inst % 3 == 0:   # quantised values -> many exact ties
            x = rng.integers(0, 3, N).astype(np.float32)
            Y = rng.integers(0, 3, M).astype(np.float32)
        else:
            x = rng.standard_normal(N).astype(np.float32)
            Y = rng.standard_normal(M).astype(np.float32)
        bc, be, brow = _brute(brute_lib, x, Y, fma)
        r = oracle_mod.sdtw(x, Y, fma=fma, last_rows=True)
        assert np.array_equal(r["last_rows"][0], brow), (inst, N, M)
        assert r["cost"][0] == bc and r["end"][0] == be


@pytest.mark.parametrize("fma", [True, False])
def test_brute_force_full_6x12(oracle_mod, brute_lib, fma):
    """The largest size of config 1's brute-force check (6 x 12)."""
    for inst in range(20):
        rng = np.random.default_rng(1200 + inst)
        x = rng.standard_normal(6).astype(np.float32)
        Y = rng.standard_normal(12).astype(np.float32)
        bc, be, brow = _brute(brute_lib, x, Y, fma)
        r = oracle_mod.sdtw(x, Y, fma=fma, last_rows=True)
        assert np.array_equal(r["last_rows"][0], brow)
        assert r["cost"][0] == bc and r["end"][0] == be


@pytest.mark.parametrize("fma", [True, False])
def test_closed_form_single_row(oracle_mod, fma):
    """N=1: cost = min_j fl((x0-yj)^2), end = first argmin, start = end."""
    rng = np.random.default_rng(11)
    for _ in range(20):
        x = rng.standard_normal(1).astype(np.float32)
        Y = rng.standard_normal(int(rng.integers(1, 300))).astype(np.float32)
        vals = np.array([cell_f32(x[0], y, 0.0, fma) for y in Y], np.float32)
        r = oracle_mod.sdtw(x, Y, fma=fma, start=True)
        assert r["cost"][0] == vals.min()
        assert r["end"][0] == int(np.argmin(vals))
        assert r["start"][0] == r["end"][0]


@pytest.mark.parametrize("fma", [True, False])
def test_closed_form_single_column(oracle_mod, fma):
    """M=1: cost = left fold of (x_i - y0)^2 down the only column, end = start = 0."""
    rng = np.random.default_rng(12)
    for _ in range(10):
        x = rng.standard_normal(int(rng.integers(1, 200))).astype(np.float32)
        Y = rng.standard_normal(1).astype(np.float32)
        r = oracle_mod.sdtw(x, Y, fma=fma, start=True)
        assert r["cost"][0] == fold_f32(x, Y[0], fma)
        assert r["end"][0] == 0 and r["start"][0] == 0


@pytest.mark.parametrize("fma", [True, False])
def test_constant_reference(oracle_mod, fma):
    """Constant reference c: every column ties, cost = fold of (x_i-c)^2, end 0 (smallest index)."""
    rng = np.random.default_rng(13)
    x = rng.standard_normal(40).astype(np.float32)
    Y = np.full(57, np.float32(0.3), np.float32)
    r = oracle_mod.sdtw(x, Y, fma=fma, start=True)
    assert r["cost"][0] == fold_f32(x, Y[0], fma)
    assert r["end"][0] == 0 and r["start"][0] == 0


@pytest.mark.parametrize("stretch", [1, 2, 3])
def test_embedding_and_integer_stretch(oracle_mod, stretch):
    """A query cut from the reference (each sample repeated k times) scores 0 at s+L-1, start s."""
    from datagen import embed_queries
    rng = np.random.default_rng(7)
    Y = rng.standard_normal(3000).astype(np.float32)
    Q, starts = embed_queries(Y, Z=6, N=300, seed=7, stretch=stretch)
    for fma in (True, False):
        r = oracle_mod.sdtw(Q, Y, fma=fma, start=True)
        assert np.all(r["cost"] == 0.0)
        assert np.array_equal(r["end"], starts + 300 - 1)
        assert np.array_equal(r["start"], starts)


def test_fractional_stretch(oracle_mod):
    """Resampling a cut at constant rate 1/2.5 with floor indexing keeps (0, s+L-1, s)."""
    rng = np.random.default_rng(7)
    Y = rng.standard_normal(4000).astype(np.float32)
    s, L = 1234, 300
    idx = np.floor(np.arange(int(L * 2.5)) / 2.5).astype(np.int64)
    q = Y[s + idx]
    r = oracle_mod.sdtw(q, Y, fma=True, start=True)
    assert r["cost"][0] == 0.0 and r["end"][0] == s + L - 1 and r["start"][0] == s


def test_general_stretch_is_not_invariant(oracle_mod):
    """Stretching an arbitrary (non-embedded) query changes its cost."""
    rng = np.random.default_rng(8)
    Y = rng.standard_normal(3000).astype(np.float32)
    q = rng.standard_normal(200).astype(np.float32)
    a = oracle_mod.sdtw(q, Y)["cost"][0]
    b = oracle_mod.sdtw(np.repeat(q, 2), Y)["cost"][0]
    assert b > a


@pytest.mark.parametrize("fma", [True, False])
def test_reference_prefix_and_extension(oracle_mod, fma):
    """Last-row cells at columns < M' are identical on Y[:M']: the prefix result is the
    prefix min of the full last row, and extending the reference never increases the cost."""
    rng = np.random.default_rng(14)
    x = rng.standard_normal(50).astype(np.float32)
    Y = rng.standard_normal(900).astype(np.float32)
    full = oracle_mod.sdtw(x, Y, fma=fma, last_rows=True)
    row = full["last_rows"][0]
    prev_cost = np.float32(np.inf)
    for Mp in (1, 7, 100, 333, 899, 900):
        r = oracle_mod.sdtw(x, Y[:Mp], fma=fma, last_rows=True)
        assert np.array_equal(r["last_rows"][0], row[:Mp])
        assert r["cost"][0] == row[:Mp].min() and r["end"][0] == int(np.argmin(row[:Mp]))
        assert r["cost"][0] <= prev_cost
        prev_cost = r["cost"][0]


@pytest.mark.parametrize("fma", [True, False])
def test_start_validity_restricted_dp(oracle_mod, brute_lib, fma):
    """A DP restricted to start exactly at s reaches exactly the cost at end."""
    for inst in range(120):
        rng = np.random.default_rng(3000 + inst)
        N = int(rng.integers(1, 25))
        M = int(rng.integers(1, 80))
        if inst % 2:
            x = rng.integers(0, 4, N).astype(np.float32)
            Y = rng.integers(0, 4, M).astype(np.float32)
        else:
            x = rng.standard_normal(N).astype(np.float32)
            Y = rng.standard_normal(M).astype(np.float32)
        r = oracle_mod.sdtw(x, Y, fma=fma, start=True)
        got = _restricted(brute_lib, x, Y, fma, r["start"][0], r["end"][0])
        assert got == r["cost"][0], (inst, got, r["cost"][0])
        # and no start strictly before... every other start is >= cost (sanity)
        assert r["start"][0] <= r["end"][0]


def test_walkback_equals_forward_start(oracle_mod):
    """The paper's walk-back over the full matrix equals the forward-propagated start."""
    for inst in range(200):
        rng = np.random.default_rng(4000 + inst)
        N = int(rng.integers(1, 30))
        M = int(rng.integers(1, 60))
        if inst % 2:
            x = rng.integers(0, 3, N).astype(np.float32)
            Y = rng.integers(0, 3, M).astype(np.float32)
        else:
            x = rng.standard_normal(N).astype(np.float32)
            Y = rng.standard_normal(M).astype(np.float32)
        for fma in (True, False):
            D, S = oracle_mod.sdtw_full(x, Y, fma=fma)
            r = oracle_mod.sdtw(x, Y, fma=fma, start=True)
            assert r["cost"][0] == D[-1].min() and r["end"][0] == int(np.argmin(D[-1]))
            assert oracle_mod.walkback(D, r["end"][0]) == r["start"][0] == S[-1, r["end"][0]]


def test_fp64_definition_accuracy(oracle_mod):
    """fp32 result within the fp32 error bound of the fp64 definition."""
    for inst in range(6):
        rng = np.random.default_rng(5000 + inst)
        x = rng.standard_normal(40).astype(np.float32)
        Y = rng.standard_normal(250).astype(np.float32)
        c64, e64, row64 = dp_f64(x, Y)
        for fma in (True, False):
            r = oracle_mod.sdtw(x, Y, fma=fma, last_rows=True)
            assert abs(float(r["cost"][0]) - c64) <= 1e-5 * max(c64, 1e-30)
            assert np.allclose(r["last_rows"][0], row64, rtol=1e-5, atol=0)
            # end agrees unless the fp64 last row has a near-tie at the fp32 end
            assert r["end"][0] == e64 or row64[r["end"][0]] <= c64 * (1 + 1e-5)


def test_fma_vs_nofma_drift(oracle_mod):
    from datagen import nanopore_queries, nanopore_reference
    Y = oracle_mod.znorm(nanopore_reference(20000, 9)[None])[0]
    Q = oracle_mod.znorm(nanopore_queries(4, 500, 20000, 9))
    a = oracle_mod.sdtw(Q, Y, fma=True)
    b = oracle_mod.sdtw(Q, Y, fma=False)
    rel = np.abs(a["cost"] - b["cost"]) / np.maximum(a["cost"], 1e-30)
    assert rel.max() < 1e-5


def test_reversal(oracle_mod):
    """cost(rev X, rev Y) ~ cost (different fold order); end_rev = M-1-start."""
    rng = np.random.default_rng(15)
    for _ in range(10):
        x = rng.standard_normal(30).astype(np.float32)
        Y = rng.standard_normal(400).astype(np.float32)
        f = oracle_mod.sdtw(x, Y, start=True)
        b = oracle_mod.sdtw(x[::-1].copy(), Y[::-1].copy(), start=True)
        assert abs(f["cost"][0] - b["cost"][0]) <= 1e-5 * f["cost"][0]
        assert b["end"][0] == 400 - 1 - f["start"][0]
        assert b["start"][0] == 400 - 1 - f["end"][0]


def test_nonnegative(oracle_mod):
    rng = np.random.default_rng(16)
    Q = rng.standard_normal((8, 20)).astype(np.float32) * 5
    Y = rng.standard_normal(300).astype(np.float32)
    assert np.all(oracle_mod.sdtw(Q, Y)["cost"] >= 0)


# --------------------------------------------------------------- normaliser
def test_normalizer_fixture(oracle_mod):
    g = _gold("normalizer_example.json")
    z = oracle_mod.znorm(np.array(g["series"], np.float32))
    assert np.allclose(z, g["z"], atol=1e-7)
    z0 = oracle_mod.znorm(np.array(g["constant_series"], np.float32))
    assert np.array_equal(z0, np.array(g["constant_z"], np.float32))
    # population std: mean 2, std sqrt(2/3)
    x = np.array(g["series"], np.float64)
    assert np.isclose(np.sqrt((x ** 2).mean() - x.mean() ** 2), g["std"], atol=1e-7)


def test_normalizer_stats_recheck(oracle_mod):
    """|mean| <= 1e-5, |std-1| <= 1e-4 by an fp64 recheck."""
    from datagen import nanopore_queries
    Q = nanopore_queries(64, 2000, 50000, 21)
    Z = oracle_mod.znorm(Q).astype(np.float64)
    assert np.all(np.abs(Z.mean(axis=1)) <= 1e-5)
    assert np.all(np.abs(Z.std(axis=1) - 1.0) <= 1e-4)
    # exact fp64 definition, one rounding: compare with numpy fp64
    Qd = Q.astype(np.float64)
    mu = Qd.mean(axis=1, keepdims=True)
    sd = np.sqrt((Qd ** 2).mean(axis=1, keepdims=True) - mu ** 2)
    ref = ((Qd - mu) / sd).astype(np.float32)
    assert np.max(np.abs(ref.astype(np.float64) - Z)) <= 2.4e-7


def test_normalizer_exact_sums_order_free(oracle_mod):
    """Reading G8: the sums are exact, rounded once, so (a) permuting a
    series permutes z bit for bit -- a plain sequential fp64 accumulation fails this on
    most of these series (checked below, so the pin discriminates) -- and (b) z equals the
    value computed from EXACT RATIONAL sums (fractions.Fraction, rounded once to fp64 by
    float()), independently of math.fsum."""
    from fractions import Fraction
    from datagen import nanopore_queries
    Q = nanopore_queries(24, 2000, 50000, 23)
    rng = np.random.default_rng(23)
    perm = rng.permutation(Q.shape[1])
    z = oracle_mod.znorm(Q)
    zp = oracle_mod.znorm(Q[:, perm])
    assert np.array_equal(zp.view(np.uint32), z[:, perm].view(np.uint32))
    naive_differs = 0
    for q in range(Q.shape[0]):
        a = b = 0.0
        for v, w in zip(Q[q].astype(np.float64), Q[q, perm].astype(np.float64)):
            a += v * v
            b += w * w
        naive_differs += a != b
    assert naive_differs >= 4
    for q in range(4):
        x = Q[q].astype(np.float64)
        n = x.shape[0]
        s = float(sum(Fraction(v) for v in x))
        s2 = float(sum(Fraction(v) * Fraction(v) for v in x))
        mean = s / n
        ex2 = s2 / n
        sd = np.sqrt(ex2 - mean * mean)
        ref = ((x - mean) / sd).astype(np.float32)
        assert np.array_equal(ref.view(np.uint32), z[q].view(np.uint32)), q


def test_normalizer_affine_invariance(oracle_mod):
    rng = np.random.default_rng(22)
    x = rng.standard_normal((10, 777)).astype(np.float32)
    for a, b in ((3.0, 5.0), (0.25, -90.0), (12.0, 90.0)):
        y = (np.float32(a) * x + np.float32(b)).astype(np.float32)
        assert np.max(np.abs(oracle_mod.znorm(y) - oracle_mod.znorm(x))) <= 1e-4


def test_normalizer_degenerate(oracle_mod):
    x = np.full((3, 100), 93.25, np.float32)
    x[1] = 0.0
    assert np.all(oracle_mod.znorm(x) == 0.0)


def test_normalized_end_to_end_embedding(oracle_mod):
    """With z-normalisation on, an embedded cut still ends at the right column (tolerance mode)."""
    from datagen import nanopore_reference
    Y = nanopore_reference(20000, 3)
    Yn = oracle_mod.znorm(Y[None])[0]
    s, L = 4321, 400
    r = oracle_mod.sdtw_normalized(Y[s:s + L][None], Y)
    # a per-query z-norm of a cut differs from the globally normalised reference, so the
    # cost is small but not 0; the end column must still be found
    assert r["end"][0] == s + L - 1
    raw = oracle_mod.sdtw(Yn[s:s + L][None], Yn)
    assert raw["cost"][0] == 0.0
