"""GPU parity of the packed-half precision (SDTW_OPT_PRECISION=16, SURVEY.md §8(f) NEXT-1:
the paper's __half2 cells) against the oracle's half mode (every op rounded to
binary16; pinned in tests/test_oracle16_pins.py).  Raw mode: cost bit-exact, end exact or a
tie in the oracle's (half) last row."""
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


def _gpu16(Q, Y, **opts):
    kw = dict(OPT_NORMALIZE=0, OPT_PRECISION=16)
    kw.update(opts)
    with sd.options(**kw):
        sd.set_reference(torch.as_tensor(Y, device=DEV))
        c, e = sd.batch(torch.as_tensor(np.ascontiguousarray(Q), device=DEV))
    return c.cpu().numpy(), e.cpu().numpy()


def _check(Q, Y, c, e, idx=None):
    ref = oracle.sdtw(Q if idx is None else Q[idx], Y, half=True, last_rows=True)
    cc = c if idx is None else c[idx]
    ee = e if idx is None else e[idx]
    assert np.array_equal(cc.view(np.uint32), ref["cost"].view(np.uint32)), (cc[:4], ref["cost"][:4])
    for k in np.nonzero(ee != ref["end"])[0]:
        assert ref["last_rows"][k, ee[k]] == ref["cost"][k], (k, ee[k], ref["end"][k])


@pytest.mark.parametrize("W", [14, 30, 62])
@pytest.mark.parametrize("Z,N,M", [(8, 64, 4096), (5, 300, 2000), (3, 1, 500), (3, 40, 1), (3, 90, 60),
                                   (4, 257, 3000)])
def test_half_bit_exact_small(Z, N, M, W):
    Q, Y = _inputs(Z, N, M, 40 + N)
    c, e = _gpu16(Q, Y, OPT_SEGMENT_W=W)
    _check(Q, Y, c, e)


def test_half_schedules_identical():
    Q, Y = _inputs(8, 200, 20_000, 41)
    base = _gpu16(Q, Y)
    for opts in (dict(OPT_LANES=2), dict(OPT_LANES=8, OPT_CHUNK=32), dict(OPT_SCHED=2, OPT_SEGMENTS=3),
                 dict(OPT_SEGMENT_W=62, OPT_LANES=3)):
        got = _gpu16(Q, Y, **opts)
        assert np.array_equal(got[0].view(np.uint32), base[0].view(np.uint32)) and np.array_equal(got[1], base[1])


def test_half_persistent_sampled():
    Q, Y = _inputs(300, 500, 100_000, 42)
    c, e = _gpu16(Q, Y)
    idx = np.array([0, 7, 150, 299])
    _check(Q, Y, c, e, idx)


def test_half_ragged():
    rng = np.random.default_rng(43)
    lens = rng.integers(20, 400, 10)
    Y = oracle.znorm(nanopore_reference(5000, 43)[None])[0]
    qs = [oracle.znorm(nanopore_queries(1, int(n), 5000, 430 + k))[0] for k, n in enumerate(lens)]
    off = np.zeros(11, np.int64)
    off[1:] = np.cumsum(lens)
    with sd.options(OPT_NORMALIZE=0, OPT_PRECISION=16):
        sd.set_reference(Y)
        c, e = sd.batch_ragged(np.concatenate(qs), off)
    for k in range(10):
        r = oracle.sdtw(qs[k][None], Y, half=True)
        assert c[k] == r["cost"][0] and e[k] == r["end"][0], k


def test_half_close_to_fp32_end_to_end():
    """Normalised, half vs the fp32 oracle: relative cost error within the fp16 tolerance."""
    Yraw = nanopore_reference(30_000, 44)
    Qraw = nanopore_queries(16, 1000, 30_000, 44)
    with sd.options(OPT_PRECISION=16):
        sd.set_reference(Yraw)
        c, e = sd.batch(Qraw)
    ref = oracle.sdtw(oracle.znorm(Qraw), oracle.znorm(Yraw[None])[0])
    rel = np.abs(c.astype(np.float64) - ref["cost"]) / np.maximum(ref["cost"], 1e-3)
    assert np.all(rel < 3e-2), rel


def test_half_rejects_traceback_and_clusters():
    with sd.options(OPT_PRECISION=16):
        sd.set_reference(np.zeros(100, np.float32))
        with pytest.raises(sd.SdtwError):
            sd.traceback(np.ones((2, 10), np.float32))
        with sd.options(OPT_CLUSTER=2):
            with pytest.raises(sd.SdtwError):
                sd.batch(np.ones((2, 10), np.float32))


def test_half_speculative_small_batch_and_recompute():
    """Speculative segments in packed half: a small batch bit-exact against
    the half oracle and identical to sequential segments; queries copying the reference
    across segment boundaries force failed corrections and recomputation, still exact."""
    Q, Y = _inputs(6, 300, 200_000, 45)
    c, e = _gpu16(Q, Y, OPT_SCHED=3)
    _check(Q, Y, c, e)
    c2, e2 = _gpu16(Q, Y, OPT_SCHED=2, OPT_SEGMENTS=3)
    assert np.array_equal(c.view(np.uint32), c2.view(np.uint32)) and np.array_equal(e, e2)
    M, N, Sg = 100_000, 1500, 8
    Y = oracle.znorm(nanopore_reference(M, 46)[None])[0]
    Pr = -(-M // 960)
    bounds = [(s * Pr // Sg) * 960 for s in range(1, 4)]
    Q = np.stack([Y[b - 200:b + N - 200] for b in bounds]).astype(np.float32)
    c, e = _gpu16(Q, Y, OPT_SCHED=3, OPT_LANES=1, OPT_SPEC_ROUNDS=1, OPT_SEGMENTS=Sg)
    assert sd.spec_recomputed() == len(bounds)
    _check(Q, Y, c, e)
