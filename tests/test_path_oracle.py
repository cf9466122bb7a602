"""Pins of the oracle's full warp path (the paper's walk-back,
P:L35, emitted as per-row column ranges).  CPU only.

* the left fold of the cell costs along the path, computed with an exact-rational FMA
  (tests/_exact.py, independent of the oracle's fmaf), equals the cost bit for bit --
  a dropped or extra cell, a wrong column or a wrong row fails it;
* shape: monotone, connected, from (0, start) to (N-1, end), start == the forward S;
* brute force: the path cost is the minimum over all warp paths (tests/pins/brute.c);
* closed forms: a query cut from the reference follows the diagonal, a k-times
  stretched cut moves down k rows per column (tie priority diag > up > left);
* the window reduction the CUDA path uses: the DP restricted to reference columns
  [start, end] with a free start reproduces the full-matrix path exactly.
"""
import numpy as np
import pytest

from tests._exact import cell_f32


def _cases(seed0, n):
    for inst in range(n):
        rng = np.random.default_rng(seed0 + inst)
        N = int(rng.integers(1, 11))
        M = int(rng.integers(1, 31))
        if inst % 3 == 0:   # quantised -> exact ties everywhere
            x = rng.integers(0, 3, N).astype(np.float32)
            Y = rng.integers(0, 3, M).astype(np.float32)
        else:
            x = rng.standard_normal(N).astype(np.float32)
            Y = rng.standard_normal(M).astype(np.float32)
        yield inst, x, Y


def _cells(lo, hi):
    for i in range(len(lo)):
        for j in range(int(lo[i]), int(hi[i]) + 1):
            yield i, j


def _fold(x, Y, lo, hi, fma):
    v = None
    for i, j in _cells(lo, hi):
        v = cell_f32(x[i], Y[j], np.float32(0.0) if v is None else v, fma)
    return np.float32(v)


@pytest.mark.parametrize("fma", [True, False])
def test_path_fold_equals_cost_and_shape(oracle_mod, fma):
    for inst, x, Y in _cases(3001, 200):
        cost, end, start, lo, hi = oracle_mod.sdtw_path(x, Y, fma=fma)
        N = x.shape[0]
        assert lo[0] == start and hi[N - 1] == end, inst
        assert np.all(lo <= hi)
        assert np.all((lo[1:] == hi[:-1]) | (lo[1:] == hi[:-1] + 1)), inst   # down or diagonal
        assert _fold(x, Y, lo, hi, fma) == cost, inst


@pytest.mark.parametrize("fma", [True, False])
def test_path_is_optimal_brute_force(oracle_mod, brute_lib, fma):
    from tests.test_oracle_pins import _brute
    for inst, x, Y in _cases(3301, 60):
        if x.shape[0] > 6 or Y.shape[0] > 12:
            x, Y = x[:6], Y[:12]
        bc, be, _ = _brute(brute_lib, x, Y, fma)
        cost, end, start, lo, hi = oracle_mod.sdtw_path(x, Y, fma=fma)
        assert cost == bc and end == be
        assert _fold(x, Y, lo, hi, fma) == bc


def test_path_walkback_start_consistent(oracle_mod):
    for inst, x, Y in _cases(3401, 100):
        D, S = oracle_mod.sdtw_full(x, Y)
        end = int(np.argmin(D[-1]))
        lo, hi = oracle_mod.walkback_path(D, end)
        assert lo[0] == oracle_mod.walkback(D, end) == S[-1, end]


@pytest.mark.parametrize("k", [1, 2, 3])
def test_path_embedded_and_stretched_cut(oracle_mod, k):
    rng = np.random.default_rng(7)
    Y = rng.standard_normal(400).astype(np.float32)
    s, L = 123, 40
    x = np.repeat(Y[s:s + L], k)
    for fma in (True, False):
        cost, end, start, lo, hi = oracle_mod.sdtw_path(x, Y, fma=fma)
        assert cost == 0.0 and start == s and end == s + L - 1
        want = s + np.arange(L * k) // k
        assert np.array_equal(lo, want) and np.array_equal(hi, want)


def test_path_tie_priority_fixture(oracle_mod):
    """x = y = [1, 1]: every D is 0; from (1,1) the diag predecessor wins the tie."""
    D, _ = oracle_mod.sdtw_full(np.ones(2, np.float32), np.ones(2, np.float32))
    assert np.all(D == 0)
    lo, hi = oracle_mod.walkback_path(D, 1)
    assert list(lo) == [0, 1] and list(hi) == [0, 1]
    lo, hi = oracle_mod.walkback_path(D, 0)          # column 0: only "up" exists
    assert list(lo) == [0, 0] and list(hi) == [0, 0]


@pytest.mark.parametrize("fma", [True, False])
def test_path_window_reduction(oracle_mod, fma):
    """Restricting the DP to columns [start, end] (free start, +inf left edge) gives the same
    end and the same path: the reduction sdtw_path's CUDA kernels rely on."""
    for inst, x, Y in _cases(3501, 200):
        cost, end, start, lo, hi = oracle_mod.sdtw_path(x, Y, fma=fma)
        wc, we, ws, wlo, whi = oracle_mod.sdtw_path(x, Y[start:end + 1], fma=fma)
        assert wc == cost and we == end - start and ws == 0, inst
        assert np.array_equal(wlo + start, lo) and np.array_equal(whi + start, hi), inst
