"""Pins of the uint8-codebook oracle (§Discussion P:L165;
DESIGN.md §16, readings G18-G21) against things other than itself:

* the codebook's order statistics against counting (no sort), and the clip extremes;
* the code formula against hand-computed fixtures (exact binary fractions), monotonicity and
  the clamp of outliers;
* the integer DP against brute-force enumeration of every warp path on tiny inputs, with
  and without INF pruning (the path value composes the cell maps; the min over paths equals
  the DP because every cell map is monotone);
* the unpruned integer DP against the (independently pinned) fp32 oracle on integer-valued
  inputs small enough that every fp32 operation is exact;
* pruning invariants: tau >= 255 is no pruning, the cost never increases with tau, an exact
  code slice survives tau = 0, codes that never match give INF;
* the accuracy metric of the approximation on nanopore-like workloads: the end index of the
  uint8 path against the fp32 end (reported, bounded here loosely).
"""
import itertools

import numpy as np
import pytest

import oracle

INF = oracle.Q8_INF


# ------------------------------------------------------------------ codebook + codes
def test_codebook_is_the_order_statistic_by_counting():
    rng = np.random.default_rng(11)
    for M, clip in [(1, 1000), (2, 0), (7, 200_000), (1000, 1000), (5003, 50_000), (20_000, 1000)]:
        Y = np.round(rng.normal(size=M) * 8).astype(np.float32) / 8     # many ties
        lo, hi = oracle.codebook(Y, clip)
        k = (clip * (M - 1)) // 1_000_000
        for v, r in [(lo, k), (hi, M - 1 - k)]:
            assert np.sum(Y < v) <= r < np.sum(Y <= v), (M, clip, v, r)
    Y = rng.normal(size=999).astype(np.float32)
    lo, hi = oracle.codebook(Y, 0)
    assert lo == Y.min() and hi == Y.max()


def test_quantize_fixtures():
    # lo = 0, hi = 255: scale 1, code = floor(v + 0.5) clamped
    v = np.array([-3.0, 0.0, 0.25, 0.49, 0.5, 1.5, 127.5, 254.5, 255.0, 300.0], np.float32)
    assert oracle.quantize(v, 0.0, 255.0).tolist() == [0, 0, 0, 0, 1, 2, 128, 255, 255, 255]
    # lo = -1, hi = 1: scale 127.5; 0 -> floor(128.0) = 128; the ends map to 0 / 255
    v = np.array([-1.0, -0.5, 0.0, 0.5, 1.0, -7.0, 9.0], np.float32)
    # -0.5 -> 63.75 + 0.5 = 64.25 -> 64; 0.5 -> 191.25 + 0.5 -> 191
    assert oracle.quantize(v, -1.0, 1.0).tolist() == [0, 64, 128, 191, 255, 0, 255]
    # degenerate codebook
    assert oracle.quantize(np.array([1.0, 2.0], np.float32), 3.0, 3.0).tolist() == [0, 0]


def test_quantize_monotone_and_uniform():
    rng = np.random.default_rng(3)
    v = np.sort(rng.normal(size=5000).astype(np.float32))
    c = oracle.quantize(v, -2.5, 2.5).astype(int)
    assert np.all(np.diff(c) >= 0)
    assert c[v <= -2.5].max(initial=0) == 0 and c[v >= 2.5].min(initial=255) == 255
    # equal-width levels: every interior level is hit by a uniform sweep, each about equally
    u = np.linspace(-2.5, 2.5, 255 * 200 + 1, dtype=np.float32)
    h = np.bincount(oracle.quantize(u, -2.5, 2.5), minlength=256)
    assert h[0] > 0 and h[255] > 0 and np.all(h[1:255] > 150) and np.all(h[1:255] < 250)


# ------------------------------------------------------------------ DP vs brute force
def _cell(t, m, tau):
    if tau >= 0 and abs(t) > tau:
        return INF
    return min(t * t + m, INF)


def _brute(x, y, tau):
    """min over every warp path (start anywhere in row 0, steps down / right / diagonal, end
    in row N-1) of the composed cell maps, and the smallest end column attaining it."""
    N, M = len(x), len(y)
    best = {}

    def walk(i, j, v):
        v = _cell(int(x[i]) - int(y[j]), v, tau)
        if i == N - 1:
            best[j] = min(best.get(j, INF + 1), v)
        if i + 1 < N:
            walk(i + 1, j, v)
        if j + 1 < M:
            walk(i, j + 1, v)
        if i + 1 < N and j + 1 < M:
            walk(i + 1, j + 1, v)

    for j0 in range(M):
        walk(0, j0, 0)
    cost = min(best.values())
    return cost, min(j for j, v in best.items() if v == cost)


@pytest.mark.parametrize("tau", [-1, 0, 2, 5, 255])
def test_dp_equals_brute_force(tau):
    rng = np.random.default_rng(100 + tau)
    for _ in range(120):
        N, M = int(rng.integers(1, 5)), int(rng.integers(1, 7))
        hi = int(rng.choice([4, 12, 255]))
        x = rng.integers(0, hi + 1, N).astype(np.uint8)
        y = rng.integers(0, hi + 1, M).astype(np.uint8)
        r = oracle.sdtw_q8(x, y, tau)
        c, e = _brute(x, y, tau)
        assert (int(r["cost"][0]), int(r["end"][0])) == (c, e), (x, y, tau)


def test_unpruned_equals_fp32_oracle_on_exact_integers():
    """Codes < 2^4: N * 15^2 < 2^24, so the fp32 oracle's operations are exact on these
    integer-valued inputs (both FMA modes); the integer DP must give the same cost and end."""
    rng = np.random.default_rng(7)
    for N, M in [(1, 9), (5, 40), (30, 300), (200, 700)]:
        x = rng.integers(0, 16, (3, N)).astype(np.uint8)
        y = rng.integers(0, 16, M).astype(np.uint8)
        r = oracle.sdtw_q8(x, y, -1)
        for fma in (False, True):
            f = oracle.sdtw(x.astype(np.float32), y.astype(np.float32), fma=fma)
            assert np.array_equal(r["cost"], f["cost"].astype(np.int64)), (N, M)
            assert np.array_equal(r["end"], f["end"])


# ------------------------------------------------------------------ pruning invariants
def test_pruning_invariants():
    rng = np.random.default_rng(5)
    y = rng.integers(0, 256, 3000).astype(np.uint8)
    x = rng.integers(0, 256, (6, 40)).astype(np.uint8)
    base = oracle.sdtw_q8(x, y, -1)
    same = oracle.sdtw_q8(x, y, 255)
    assert np.array_equal(base["cost"], same["cost"]) and np.array_equal(base["end"], same["end"])
    prev = None
    for tau in [0, 1, 3, 8, 20, 60, 128, 254]:
        c = oracle.sdtw_q8(x, y, tau)["cost"]
        assert np.all(c >= base["cost"])
        if prev is not None:
            assert np.all(c <= prev)                      # pruning less never costs more
        prev = c
    # an exact slice survives tau = 0 with cost 0 at its end
    s = 1234
    r = oracle.sdtw_q8(y[s:s + 25], y, 0)
    assert r["cost"][0] == 0 and r["end"][0] == s + 24
    # codes absent from the reference: every path pruned at tau = 0
    y2 = (rng.integers(0, 128, 500) * 2).astype(np.uint8)        # even codes
    r = oracle.sdtw_q8(np.array([[1, 3, 5]], np.uint8), y2, 0)
    assert r["cost"][0] == INF and r["end"][0] == 0


def test_embedding_is_exact():
    rng = np.random.default_rng(9)
    y = rng.integers(0, 256, 5000).astype(np.uint8)
    for s, L in [(0, 30), (777, 60), (4970, 30)]:
        r = oracle.sdtw_q8(y[s:s + L], y, -1)
        assert r["cost"][0] == 0 and r["end"][0] == s + L - 1


# ------------------------------------------------------------------ accuracy metric
def test_end_agreement_with_fp32_on_nanopore_cuts():
    """The approximation's accuracy metric: for queries cut from the
    reference, the uint8 end index against the fp32 end.  Reported in DESIGN.md §16 and by
    the bench; bounded loosely here so that a broken codebook fails."""
    from datagen import nanopore_queries, nanopore_reference
    M = 60_000
    Y = nanopore_reference(M, 21)
    Q = nanopore_queries(24, 400, M, 21)
    f = oracle.sdtw_normalized(Q, Y)
    for tau in (-1, 96):                       # 96 codes ~ 2.4 normalised units (the bench's)
        q = oracle.sdtw_q8_normalized(Q, Y, tau=tau)
        d = np.abs(q["end"] - f["end"])
        assert np.mean(d <= 8) >= 0.6, (tau, d)
        assert np.all(q["cost"] < INF)
    # a harsh threshold prunes every path of most queries: one far sample kills them all
    q = oracle.sdtw_q8_normalized(Q, Y, tau=8)
    assert np.mean(q["cost"] == INF) > 0.5
