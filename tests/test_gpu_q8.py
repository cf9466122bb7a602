"""GPU parity of the uint8-codebook variant (SDTW_OPT_PRECISION=8 / sdtw_batch_q8, SURVEY.md
§8(f) NEXT-3; §Discussion) against the oracle
(oracle.codebook / quantize / sdtw_q8, pinned in tests/test_oracle_q8_pins.py):

* the codebook (two exact order statistics by radix select on the GPU) and the codes: bit-exact;
* the integer DP with and without INF pruning: cost (int32) and end exact -- integer work,
  no tolerance -- across segment widths, lane counts and the sequential, persistent and
  speculative schedules (incl. forced recomputation), ragged batches, sampled queries of
  the paper's batch shape;
* the scaled fp32 cost of sdtw_batch at OPT_PRECISION=8; argument errors.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle  # noqa: E402
import paper_2403_06931_b200 as sd  # noqa: E402
from datagen import nanopore_queries, nanopore_reference  # noqa: E402

DEV = torch.device("cuda", 0)


def _inputs(Z, N, M, seed):
    Y = oracle.znorm(nanopore_reference(M, seed)[None])[0]
    Q = oracle.znorm(nanopore_queries(Z, N, M, seed))
    return Q, Y


def _gpu8(Q, Y, tau=-1, **opts):
    kw = dict(OPT_NORMALIZE=0, OPT_Q8_PRUNE=tau)
    kw.update(opts)
    with sd.options(**kw):
        sd.set_reference(torch.as_tensor(Y, device=DEV))
        c, e = sd.batch_q8(torch.as_tensor(np.ascontiguousarray(Q), device=DEV))
    return c.cpu().numpy(), e.cpu().numpy()


def _ref(Q, Y, tau=-1, clip=1000):
    lo, hi = oracle.codebook(Y, clip)
    return oracle.sdtw_q8(oracle.quantize(Q, lo, hi), oracle.quantize(Y, lo, hi), tau)


def _check(Q, Y, c, e, tau=-1, idx=None):
    Qs = Q if idx is None else Q[idx]
    r = _ref(Qs, Y, tau)
    cc = c if idx is None else c[idx]
    ee = e if idx is None else e[idx]
    assert np.array_equal(cc.astype(np.int64), r["cost"]), (cc[:6], r["cost"][:6])
    assert np.array_equal(ee, r["end"]), (ee[:6], r["end"][:6])


# ------------------------------------------------------------------ codebook + codes
@pytest.mark.parametrize("M,clip", [(1, 1000), (2, 1000), (4096, 1000), (100_000, 1000), (100_000, 0),
                                    (77_777, 123_456), (1_000_000, 1000)])
def test_codebook_bit_exact(M, clip):
    Y = oracle.znorm(nanopore_reference(M, 3)[None])[0] if M > 2 else np.array([0.5, -2.0][:M], np.float32)
    if M == 77_777:
        Y = (np.round(Y * 16) / 16).astype(np.float32)          # heavy ties
    with sd.options(OPT_NORMALIZE=0, OPT_Q8_CLIP=clip):
        sd.set_reference(torch.as_tensor(Y, device=DEV))
        lo, hi = sd.q8_codebook()
    rlo, rhi = oracle.codebook(Y, clip)
    assert (lo, hi) == (rlo, rhi)


def test_codes_bit_exact():
    Q, Y = _inputs(4, 5000, 50_000, 5)
    with sd.options(OPT_NORMALIZE=0):
        sd.set_reference(torch.as_tensor(Y, device=DEV))
        lo, hi = sd.q8_codebook()
        X = np.concatenate([Q.ravel(), np.array([lo, hi, lo - 1, hi + 1, 0.0, -0.0, 1e30, -1e30], np.float32)])
        got = sd.quantize(torch.as_tensor(X, device=DEV)).cpu().numpy()
        got_host = sd.quantize(X)
    ref = oracle.quantize(X, lo, hi)
    assert np.array_equal(got, ref) and np.array_equal(got_host, ref)
    assert got[-8] == 0 and got[-7] == 255


# ------------------------------------------------------------------ DP parity
@pytest.mark.parametrize("W", [14, 30])
@pytest.mark.parametrize("tau", [-1, 0, 24, 96])
@pytest.mark.parametrize("Z,N,M", [(8, 64, 4096), (5, 300, 2000), (3, 1, 500), (3, 40, 1), (3, 90, 60),
                                   (4, 257, 3001)])
def test_q8_bit_exact_small(Z, N, M, tau, W):
    Q, Y = _inputs(Z, N, M, 50 + N)
    c, e = _gpu8(Q, Y, tau, OPT_SEGMENT_W=W)
    _check(Q, Y, c, e, tau)


@pytest.mark.parametrize("tau", [-1, 40])
def test_q8_schedules_identical(tau):
    Q, Y = _inputs(8, 200, 60_000, 51)
    base = _gpu8(Q, Y, tau)
    _check(Q, Y, *base, tau)
    for opts in (dict(OPT_SCHED=1), dict(OPT_LANES=2), dict(OPT_LANES=8, OPT_CHUNK=32),
                 dict(OPT_SCHED=2, OPT_SEGMENTS=3), dict(OPT_LANES=3), dict(OPT_SCHED=3),
                 dict(OPT_SEGMENT_W=30), dict(OPT_SEGMENT_W=30, OPT_SCHED=2, OPT_SEGMENTS=3)):
        got = _gpu8(Q, Y, tau, **opts)
        assert np.array_equal(got[0], base[0]) and np.array_equal(got[1], base[1]), opts


def test_q8_speculative_recompute():
    """Queries copying the reference across segment boundaries with one-round corrections:
    every correction fails and the query is recomputed from its codes -- still exact."""
    M, N, Sg = 100_000, 1500, 8
    Y = oracle.znorm(nanopore_reference(M, 56)[None])[0]
    Pr = -(-M // 960)
    bounds = [(s * Pr // Sg) * 960 for s in range(1, 4)]
    Q = np.stack([Y[b - 200:b + N - 200] for b in bounds]).astype(np.float32)
    for tau in (-1, 60):
        c, e = _gpu8(Q, Y, tau, OPT_SCHED=3, OPT_LANES=1, OPT_SPEC_ROUNDS=1, OPT_SEGMENTS=Sg)
        assert sd.spec_recomputed() == len(bounds)
        _check(Q, Y, c, e, tau)
        assert np.all(c == 0)


def test_q8_paper_shape_sampled():
    """The paper's batch shape (512 x 2,000 vs 100,000) in the bench's
    launch configuration, 12 queries checked against the oracle."""
    Q, Y = _inputs(512, 2000, 100_000, 57)
    idx = np.array([0, 1, 63, 64, 200, 255, 256, 300, 409, 450, 510, 511])
    for tau in (-1, 96):
        c, e = _gpu8(Q, Y, tau)
        _check(Q, Y, c, e, tau, idx)


def test_q8_normalised_end_to_end_and_scaled_cost():
    Yraw = nanopore_reference(30_000, 58)
    Qraw = nanopore_queries(16, 700, 30_000, 58)
    ref = oracle.sdtw_q8_normalized(Qraw, Yraw, tau=96)
    with sd.options(OPT_Q8_PRUNE=96):
        sd.set_reference(Yraw)
        c, e = sd.batch_q8(Qraw)
        with sd.options(OPT_PRECISION=8):
            cf, ef = sd.batch(Qraw)
        lo, hi = sd.q8_codebook()
    assert np.array_equal(c.astype(np.int64), ref["cost"]) and np.array_equal(e, ref["end"])
    assert (lo, hi) == (ref["lo"], ref["hi"])
    delta = (np.float64(hi) - np.float64(lo)) / 255.0
    want = (ref["cost"].astype(np.float64) * (delta * delta)).astype(np.float32)
    assert np.array_equal(cf, want) and np.array_equal(ef, e)


def test_q8_pruned_everywhere_and_long_queries():
    """Every path pruned (cost INF, end 0 -- the GPU's unclamped form canonicalised) and the
    longest pruned queries (N = 8,000) against the oracle's clamped definition."""
    Q, Y = _inputs(6, 8000, 40_000, 60)
    for tau in (0, 3, 60):
        c, e = _gpu8(Q, Y, tau)
        _check(Q, Y, c, e, tau)
    assert np.all(_gpu8(Q, Y, 0)[0] == oracle.Q8_INF)


def test_q8_ragged():
    rng = np.random.default_rng(59)
    lens = rng.integers(20, 600, 12)
    Y = oracle.znorm(nanopore_reference(40_000, 59)[None])[0]
    qs = [oracle.znorm(nanopore_queries(1, int(n), 40_000, 590 + k))[0] for k, n in enumerate(lens)]
    off = np.zeros(13, np.int64)
    off[1:] = np.cumsum(lens)
    lo, hi = oracle.codebook(Y)
    delta = (np.float64(hi) - np.float64(lo)) / 255.0
    with sd.options(OPT_NORMALIZE=0, OPT_PRECISION=8):
        sd.set_reference(Y)
        c, e = sd.batch_ragged(np.concatenate(qs), off)
    for k in range(12):
        r = _ref(qs[k][None], Y)
        assert c[k] == np.float32(np.float64(r["cost"][0]) * (delta * delta)) and e[k] == r["end"][0], k


def test_q8_errors():
    with sd.options(OPT_PRECISION=8):
        sd.set_reference(np.zeros(100, np.float32))
        with pytest.raises(sd.SdtwError):
            sd.traceback(np.ones((2, 10), np.float32))
        with pytest.raises(sd.SdtwError):
            sd.batch_q8(np.ones((1, 12_001), np.float32))
        with sd.options(OPT_Q8_PRUNE=40):                     # pruning: N <= 8,000 (sdtw_q8.cuh)
            with pytest.raises(sd.SdtwError):
                sd.batch_q8(np.ones((1, 8_001), np.float32))
        with pytest.raises(sd.SdtwError):
            sd.quantize(np.array([1.0, np.nan], np.float32))
        with sd.options(OPT_SEGMENT_W=62):                   # W = 14 or 30
            with pytest.raises(sd.SdtwError):
                sd.batch_q8(np.ones((1, 10), np.float32))
    with pytest.raises(sd.SdtwError):
        sd.set_option(sd.OPT_Q8_PRUNE, 256)
