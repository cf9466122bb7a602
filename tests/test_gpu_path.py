"""GPU parity of sdtw_path (the full warp path) against the CPU oracle.

Raw mode (inputs normalised by the oracle, OPT_NORMALIZE=0), same FMA mode on both
sides: cost bit-exact, end / start exact, the path (per-row column ranges) exact --
the oracle's walk-back over its full matrix (tests/test_path_oracle.py pins it).
Long references: the oracle runs on the window [start, end] (the reduction pinned
by test_path_window_reduction) and the path's exact-FMA fold must equal the cost.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle  # noqa: E402
import paper_2403_06931_b200 as sd  # noqa: E402
from datagen import embed_queries, nanopore_queries, nanopore_reference  # noqa: E402

DEV = torch.device("cuda", 0)


def _gpu_path(Q, Y, **opts):
    kw = dict(OPT_NORMALIZE=0)
    kw.update(opts)
    with sd.options(**kw):
        sd.set_reference(torch.as_tensor(Y, device=DEV))
        c, e, s, lo, hi = sd.path(torch.as_tensor(np.ascontiguousarray(Q), device=DEV))
    return c.cpu().numpy(), e.cpu().numpy(), s.cpu().numpy(), lo.cpu().numpy(), hi.cpu().numpy()


def _inputs(Z, N, M, seed, quantised=False):
    if quantised:
        rng = np.random.default_rng(seed)
        return rng.integers(0, 3, (Z, N)).astype(np.float32), rng.integers(0, 3, M).astype(np.float32)
    Y = oracle.znorm(nanopore_reference(M, seed)[None])[0]
    Q = oracle.znorm(nanopore_queries(Z, N, M, seed))
    return Q, Y


def _check_full(Q, Y, got, fma):
    c, e, s, lo, hi = got
    for q in range(Q.shape[0]):
        rc, re, rs, rlo, rhi = oracle.sdtw_path(Q[q], Y, fma=fma)
        assert c[q].view(np.uint32) == np.float32(rc).view(np.uint32), q
        assert e[q] == re and s[q] == rs, (q, e[q], re, s[q], rs)
        assert np.array_equal(lo[q], rlo) and np.array_equal(hi[q], rhi), q


@pytest.mark.parametrize("fma", [1, 0])
@pytest.mark.parametrize("Z,N,M,quant", [
    (8, 64, 4096, False),      # BASELINE config 1
    (6, 300, 2000, False),     # two bands of rows (256 + 44)
    (5, 257, 700, True),       # exact ties everywhere, one-row second band
    (4, 1, 500, False),        # N = 1
    (3, 40, 1, False),         # M = 1: the path is one column
    (3, 90, 60, False),        # N > M
])
def test_path_bit_exact_small(Z, N, M, quant, fma):
    Q, Y = _inputs(Z, N, M, 11 + N, quant)
    _check_full(Q, Y, _gpu_path(Q, Y, OPT_FMA=fma), bool(fma))


def test_path_host_pointers_match_device():
    Q, Y = _inputs(4, 100, 3000, 5)
    dev = _gpu_path(Q, Y)
    with sd.options(OPT_NORMALIZE=0):
        sd.set_reference(Y)
        host = sd.path(Q)
    for a, b in zip(dev, host):
        assert np.array_equal(a, np.asarray(b))


def test_path_embedded_cuts_are_diagonal():
    rng = np.random.default_rng(7)
    Y = rng.standard_normal(200_000).astype(np.float32)
    Q, starts = embed_queries(Y, Z=8, N=500, seed=7, stretch=1)
    c, e, s, lo, hi = _gpu_path(Q, Y)
    assert np.all(c == 0) and np.array_equal(s, starts)
    want = starts[:, None] + np.arange(500)[None, :]
    assert np.array_equal(lo, want) and np.array_equal(hi, want)


@pytest.mark.parametrize("N", [500, 1000])
def test_path_config5_shape_window(N):
    """BASELINE config 5 shapes (1M reference, start index on) on a sample of queries: the
    oracle on the window [start, end] reproduces cost, end and the whole path."""
    M = 1_000_000
    Q, Y = _inputs(12, N, M, 5)
    c, e, s, lo, hi = _gpu_path(Q, Y)
    for q in range(Q.shape[0]):
        a, b = int(s[q]), int(e[q])
        assert b - a + 1 <= 8 * N, "window unexpectedly wide"
        rc, re, rs, rlo, rhi = oracle.sdtw_path(Q[q], Y[a:b + 1])
        assert np.float32(rc) == c[q] and re == b - a and rs == 0, q
        assert np.array_equal(rlo + a, lo[q]) and np.array_equal(rhi + a, hi[q]), q
        assert lo[q, 0] == a and hi[q, -1] == b
        assert np.all((lo[q, 1:] == hi[q, :-1]) | (lo[q, 1:] == hi[q, :-1] + 1))


def test_path_empty_and_errors():
    with sd.options(OPT_NORMALIZE=0):
        sd.set_reference(np.zeros(10, np.float32))
        c, e, s, lo, hi = sd.path(np.zeros((0, 5), np.float32))
        assert c.shape == (0,) and lo.shape == (0, 5)
        with pytest.raises(sd.SdtwError):
            sd.path(np.full((1, 4), np.nan, np.float32))
