"""CPU pins of the exactness argument behind the speculative segments, on a
plain float32 column-by-column DP written here (no library code): for a segment with left
boundary column T,

  D_true = min(D_free, D_bnd)   cell by cell, bit for bit,

where D_free starts freely in row 0 with a +inf boundary and D_bnd takes T with no free
start -- because cell(m) = fl(fl(x-y)^2 + m) is monotone in m and commutes with min --
and once D_bnd >= D_free on a whole column it stays so on every later column."""
import numpy as np
import pytest

F32 = np.float32
INF = F32(np.inf)


def _segment(x, y, T, zrow):
    """Columns of the DP over reference y with left boundary T (len N), virtual row -1 = zrow."""
    N = len(x)
    prev = T.astype(F32)
    prev_top = F32(zrow)                       # D(-1, j-1)
    cols = []
    for yj in y.astype(F32):
        col = np.empty(N, F32)
        up = F32(zrow)                         # D(-1, j)
        for i in range(N):
            m = min(prev[i], up, prev[i - 1] if i > 0 else prev_top)
            t = F32(x[i] - yj)
            col[i] = F32(F32(t * t) + F32(m))
            up = col[i]
        cols.append(col)
        prev = col
        prev_top = F32(zrow)
    return np.array(cols)


@pytest.mark.parametrize("seed", range(6))
def test_true_dp_is_min_of_free_and_boundary_dp(seed):
    rng = np.random.default_rng(900 + seed)
    N, L = int(rng.integers(1, 12)), int(rng.integers(1, 40))
    x = rng.standard_normal(N).astype(F32)
    y = rng.standard_normal(L).astype(F32)
    T = (rng.random(N) * 4).astype(F32)
    if seed % 3 == 0:
        T[rng.integers(0, N)] = INF
    true = _segment(x, y, T, 0.0)
    free = _segment(x, y, np.full(N, INF, F32), 0.0)
    bnd = _segment(x, y, T, INF)
    assert np.array_equal(true.view(np.uint32), np.minimum(free, bnd).view(np.uint32))


@pytest.mark.parametrize("seed", range(6))
def test_domination_persists(seed):
    rng = np.random.default_rng(950 + seed)
    N, L = int(rng.integers(2, 10)), 60
    x = rng.standard_normal(N).astype(F32)
    y = rng.standard_normal(L).astype(F32)
    T = (rng.random(N) * 2).astype(F32)
    free = _segment(x, y, np.full(N, INF, F32), 0.0)
    bnd = _segment(x, y, T, INF)
    dom = np.all(bnd >= free, axis=1)
    if dom.any():
        first = int(np.argmax(dom))
        assert dom[first:].all()
        true = _segment(x, y, T, 0.0)
        assert np.array_equal(true[first:], free[first:])
