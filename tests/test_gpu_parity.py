"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bars (BASELINE.json "Agreement", SURVEY.md §8(c) agreement rule):
  * raw mode (no normalisation), same FMA mode on both sides: cost BIT-EXACT,
    end index EXACT (or a tie: the oracle's last row at the GPU's end equals the
    minimum), start index EXACT and valid.
  * end to end with normalisation on: |dcost| <= 1e-5 * cost, end by the tie rule.
Inputs are seeded nanopore-like signals (datagen), oracle-normalised and fed raw
so that the DP itself is compared bit for bit; edge shapes cover ragged tails.
Full-size configs (BASELINE configs 2/3) run in the bench's launch configuration
and are checked on sampled queries: embedded cuts (exact closed form) and the
traceback window argument (oracle on Y[start..end] must reproduce cost/end
exactly -- DESIGN.md §4).
"""
import ctypes

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


def _gpu(Q, Y, trace=False, **opts):
    kw = dict(OPT_NORMALIZE=0)
    kw.update(opts)
    with sd.options(**kw):
        sd.set_reference(torch.as_tensor(Y, device=DEV))
        Qt = torch.as_tensor(np.ascontiguousarray(Q), device=DEV)
        if trace:
            c, e, s = sd.traceback(Qt)
            return c.cpu().numpy(), e.cpu().numpy(), s.cpu().numpy()
        c, e = sd.batch(Qt)
        return c.cpu().numpy(), e.cpu().numpy(), None


def _inputs(Z, N, M, seed):
    Y = oracle.znorm(nanopore_reference(M, seed)[None])[0]
    Q = oracle.znorm(nanopore_queries(Z, N, M, seed))
    return Q, Y


def _restricted(x, Yw, fma, start, end):
    """D(N-1, end) of the DP allowed to begin only at column `start` (tests/pins/brute.c)."""
    from tests.conftest import load_brute
    L = load_brute()
    f32p = ctypes.POINTER(ctypes.c_float)
    win = np.ascontiguousarray(Yw[start:end + 1], np.float32)
    x = np.ascontiguousarray(x, np.float32)
    a = np.empty(win.shape[0], np.float32)
    b = np.empty(win.shape[0], np.float32)
    return np.float32(L.restricted_dp(x.ctypes.data_as(f32p), x.shape[0], win.ctypes.data_as(f32p), win.shape[0],
                                      int(fma), 0, end - start, a.ctypes.data_as(f32p), b.ctypes.data_as(f32p)))


def _check_exact(Q, Y, got, fma=True, trace=False, ref=None):
    c, e, s = got
    if ref is None:
        ref = oracle.sdtw(Q, Y, fma=fma, start=trace, last_rows=True)
    assert np.array_equal(c.view(np.uint32), ref["cost"].view(np.uint32)), \
        (np.nonzero(c != ref["cost"])[0][:8], c[:4], ref["cost"][:4])
    bad = np.nonzero(e != ref["end"])[0]
    for q in bad:  # ties allowed: oracle last row at the GPU end equals the minimum
        assert ref["last_rows"][q, e[q]] == ref["cost"][q], (q, e[q], ref["end"][q])
    if trace:
        same = e == ref["end"]
        assert np.array_equal(s[same], ref["start"][same])
        Q2 = np.atleast_2d(Q)
        for q in bad:  # a tied end: its start must still be valid (restricted DP reaches the cost)
            if np.isfinite(c[q]):
                assert 0 <= s[q] <= e[q], (q, s[q], e[q])
                assert _restricted(Q2[q], Y, fma, int(s[q]), int(e[q])) == c[q], (q, s[q], e[q])
    return ref


# --------------------------------------------------------------- bit-exact DP
SCHEDULES = [
    dict(),                                                  # auto
    dict(OPT_PACKED=0, OPT_SEGMENT_W=7, OPT_LANES=1),
    dict(OPT_PACKED=0, OPT_SEGMENT_W=15, OPT_LANES=2, OPT_CHUNK=16),
    dict(OPT_PACKED=0, OPT_SEGMENT_W=15, OPT_LANES=4, OPT_CLUSTER=2),
    dict(OPT_PACKED=1, OPT_SEGMENT_W=14, OPT_LANES=1, OPT_CHUNK=8),
    dict(OPT_PACKED=1, OPT_SEGMENT_W=14, OPT_LANES=3),
    dict(OPT_PACKED=1, OPT_SEGMENT_W=14, OPT_LANES=2, OPT_CLUSTER=2),
    dict(OPT_PACKED=1, OPT_SEGMENT_W=30, OPT_LANES=4, OPT_CLUSTER=2),
    dict(OPT_PACKED=1, OPT_SEGMENT_W=30, OPT_LANES=1, OPT_CLUSTER=4),
    dict(OPT_PACKED=1, OPT_SEGMENT_W=30, OPT_LANES=2, OPT_RING=128),
    dict(OPT_PACKED=1, OPT_SEGMENT_W=30, OPT_LANES=1, OPT_CLUSTER=8, OPT_CHUNK=16),
    dict(OPT_PACKED=1, OPT_SEGMENT_W=14, OPT_LANES=8, OPT_CHUNK=64),
    dict(OPT_PACKED=2, OPT_SEGMENT_W=28, OPT_LANES=4),
    dict(OPT_PACKED=2, OPT_SEGMENT_W=28, OPT_LANES=1, OPT_CLUSTER=2),
    dict(OPT_PACKED=2, OPT_SEGMENT_W=28, OPT_LANES=2, OPT_RING=256),
    dict(OPT_SCHED=2, OPT_SEGMENTS=3),                       # persistent units (3 segments per query)
    dict(OPT_SCHED=2, OPT_SEGMENTS=2, OPT_PACKED=0, OPT_SEGMENT_W=7, OPT_LANES=2),
    dict(OPT_SCHED=1),
    dict(OPT_PACKED=3, OPT_SEGMENT_W=30, OPT_LANES=4),        # dual-query, 2 chains
    dict(OPT_PACKED=3, OPT_SEGMENT_W=14, OPT_LANES=12, OPT_SCHED=2, OPT_SEGMENTS=2),
    dict(OPT_PACKED=4, OPT_SEGMENT_W=15, OPT_LANES=2),        # dual-query, 1 chain
    dict(OPT_PACKED=4, OPT_SEGMENT_W=7, OPT_LANES=1, OPT_SCHED=2, OPT_SEGMENTS=3),
]


@pytest.mark.parametrize("fma", [1, 0])
@pytest.mark.parametrize("sched", range(len(SCHEDULES)))
def test_config1_bit_exact_all_schedules(fma, sched):
    """BASELINE config 1 (8 x 64 vs 4,096): every schedule is bit-identical to the oracle."""
    Q, Y = _inputs(8, 64, 4096, 1)
    ref = oracle.sdtw(Q, Y, fma=bool(fma), start=True, last_rows=True)
    got = _gpu(Q, Y, OPT_FMA=fma, **SCHEDULES[sched])
    _check_exact(Q, Y, got, fma=bool(fma), ref=ref)
    got_t = _gpu(Q, Y, trace=True, OPT_FMA=fma, **SCHEDULES[sched])
    _check_exact(Q, Y, got_t, fma=bool(fma), trace=True, ref=ref)


@pytest.mark.parametrize("Z,N,M", [
    (1, 1, 1), (3, 1, 1000), (2, 5, 1), (4, 7, 3), (5, 33, 97), (3, 100, 50),     # N > M
    (7, 129, 4097), (2, 300, 20001), (9, 61, 12345), (1, 2000, 2000), (33, 17, 555),
])
@pytest.mark.parametrize("packed", [0, 1, 2, 3, 4])
def test_ragged_shapes_bit_exact(Z, N, M, packed):
    rng = np.random.default_rng(Z * 1000 + N * 10 + M)
    Q = rng.standard_normal((Z, N)).astype(np.float32)
    Y = rng.standard_normal(M).astype(np.float32)
    got = _gpu(Q, Y, trace=True, OPT_PACKED=packed)
    _check_exact(Q, Y, got, trace=True)
    if M >= 4000:   # several round segments per query under the persistent scheduler
        got = _gpu(Q, Y, trace=True, OPT_PACKED=packed, OPT_SCHED=2, OPT_SEGMENTS=3, OPT_LANES=1)
        _check_exact(Q, Y, got, trace=True)


def test_quantised_inputs_ties():
    """Integer-valued inputs create many exact ties: end = smallest argmin, start by priority."""
    rng = np.random.default_rng(77)
    Q = rng.integers(0, 3, (16, 40)).astype(np.float32)
    Y = rng.integers(0, 3, 3000).astype(np.float32)
    for packed in (0, 1, 2, 3, 4):
        got = _gpu(Q, Y, trace=True, OPT_PACKED=packed)
        ref = oracle.sdtw(Q, Y, start=True, last_rows=True)
        assert np.array_equal(got[0], ref["cost"])
        assert np.array_equal(got[1], ref["end"])
        assert np.array_equal(got[2], ref["start"])


@pytest.mark.parametrize("N", [500, 1000])
def test_config5_shape_traceback(N):
    """BASELINE config 5 shape (traceback on), reduced reference so the oracle is quick."""
    Q, Y = _inputs(24, N, 30000, 5)
    got = _gpu(Q, Y, trace=True)
    _check_exact(Q, Y, got, trace=True)


def test_config2_full_batch_sampled():
    """BASELINE config 2 in full (512 x 2,000 vs 100,000, default launch); oracle on 24 sampled queries;
    the one-ring-per-query schedule must give identical bits."""
    Q, Y = _inputs(512, 2000, 100_000, 2)
    c, e, _ = _gpu(Q, Y)
    c1, e1, _ = _gpu(Q, Y, OPT_SCHED=1)
    assert np.array_equal(c, c1) and np.array_equal(e, e1)
    idx = np.linspace(0, 511, 24).astype(int)
    ref = oracle.sdtw(Q[idx], Y, start=False, last_rows=True)
    _check_exact(Q[idx], Y, (c[idx], e[idx], None), ref=ref)


def test_host_pointers_match_device_pointers():
    Q, Y = _inputs(6, 80, 5000, 3)
    with sd.options(OPT_NORMALIZE=0):
        sd.set_reference(Y)             # numpy -> host pointers
        c_h, e_h = sd.batch(Q)
        c_h2, e_h2, s_h = sd.traceback(Q)
    c_d, e_d, _ = _gpu(Q, Y)
    assert isinstance(c_h, np.ndarray)
    assert np.array_equal(c_h, c_d) and np.array_equal(e_h, e_d)
    assert np.array_equal(c_h2, c_d) and np.array_equal(e_h2, e_d)


# --------------------------------------------------------------- normaliser
@pytest.mark.parametrize("Z,L", [(64, 2000), (7, 1), (5, 3), (3, 4097), (2, 100_000)])
def test_znormalize_matches_oracle(Z, L):
    """Reading G8: exact sums on both sides -> the normaliser is bit-exact (0 mismatches)."""
    Q = nanopore_queries(Z, L, max(L, 50000), 21) if L >= 64 else \
        np.random.default_rng(L).standard_normal((Z, L)).astype(np.float32) * 12 + 90
    z = sd.znormalize(torch.as_tensor(Q, device=DEV)).cpu().numpy()
    zo = oracle.znorm(Q)
    assert np.array_equal(z.view(np.uint32), zo.view(np.uint32)), np.count_nonzero(z != zo)
    zc = sd.znormalize(np.full((2, 10), 7.0, np.float32))
    assert np.all(zc == 0)


def test_normalized_end_to_end_bit_exact():
    """Normalisation inside the call (reference at set_reference, queries per batch) equals
    the oracle's normaliser followed by the oracle's DP, bit for bit (reading G8)."""
    Yraw = nanopore_reference(50_000, 4)
    Qraw = nanopore_queries(32, 1000, 50_000, 4)
    with sd.options(OPT_NORMALIZE=1):
        sd.set_reference(torch.as_tensor(Yraw, device=DEV))
        c, e = sd.batch(torch.as_tensor(Qraw, device=DEV))
    c, e = c.cpu().numpy(), e.cpu().numpy()
    Yn = oracle.znorm(Yraw[None])[0]
    Qn = oracle.znorm(Qraw)
    _check_exact(Qn, Yn, (c, e, None))


# --------------------------------------------------------------- errors
def test_errors():
    Y = np.random.default_rng(1).standard_normal(100).astype(np.float32)
    sd.release()
    with pytest.raises(sd.SdtwError) as ei:
        sd.batch(np.zeros((2, 4), np.float32))
    assert ei.value.status == sd.E_NOREF
    bad = Y.copy()
    bad[17] = np.nan
    with pytest.raises(sd.SdtwError) as ei:
        sd.set_reference(bad)
    assert ei.value.status == sd.E_NONFINITE
    sd.set_reference(Y)
    Q = np.ones((3, 10), np.float32)
    Q[1, 4] = np.inf
    out_c = torch.full((3,), -7.0, device=DEV)
    out_e = torch.full((3,), -7, dtype=torch.int64, device=DEV)
    Qd = torch.as_tensor(Q, device=DEV)
    for norm in (0, 1):
        with sd.options(OPT_NORMALIZE=norm):
            rc = sd._lib.sdtw_batch(ctypes.c_void_p(Qd.data_ptr()), 3, 10, ctypes.c_void_p(out_c.data_ptr()),
                                    ctypes.c_void_p(out_e.data_ptr()))
        assert rc == sd.E_NONFINITE
        assert torch.all(out_c == -7.0) and torch.all(out_e == -7)   # no partial results
    c, e = sd.batch(np.zeros((0, 10), np.float32))
    assert c.shape == (0,)


def test_launch_count_and_profile():
    Q, Y = _inputs(4, 64, 4096, 1)
    n0 = sd.launch_count()
    with sd.options(OPT_PROFILE=1, OPT_NORMALIZE=0):
        sd.set_reference(torch.as_tensor(Y, device=DEV))
        sd.batch(torch.as_tensor(Q, device=DEV))
        ms, launches = sd.profile()
    assert launches == 2 and ms > 0
    assert sd.launch_count() > n0


# --------------------------------------------------------------- full scale (config 3)
@pytest.mark.slow
def test_config3_full_scale_embedded_and_window(brute_lib):
    """512 x 2,000 vs 10M in the bench's default launch; checked by
    (a) embedded cuts (exact cost 0, end = s+L-1, start = s) and
    (b) the window argument: oracle on Y[start..end] reproduces cost/end bit-exactly."""
    M, N = 10_000_000, 2000
    Y = oracle.znorm(nanopore_reference(M, 3)[None])[0]
    Q = oracle.znorm(nanopore_queries(512, N, M, 3))
    Qe, starts = embed_queries(Y, 16, N, seed=3)
    Q[:16] = Qe
    c, e, _ = _gpu(Q, Y)
    ct, et, st = _gpu(Q, Y, trace=True)
    assert np.array_equal(c, ct) and np.array_equal(e, et)
    assert np.all(c[:16] == 0) and np.array_equal(e[:16], starts + N - 1) and np.array_equal(st[:16], starts)
    for q in np.linspace(16, 511, 12).astype(int):
        lo, hi = int(st[q]), int(et[q])
        win = np.ascontiguousarray(Y[lo:hi + 1])
        r = oracle.sdtw(Q[q], win, start=True)
        assert r["cost"][0] == c[q], (q, r["cost"][0], c[q])
        assert r["end"][0] == hi - lo
        # the start is valid: a DP restricted to begin exactly at column `lo` reaches the cost
        a = np.empty(win.shape[0], np.float32)
        b = np.empty(win.shape[0], np.float32)
        f32p = ctypes.POINTER(ctypes.c_float)
        x = np.ascontiguousarray(Q[q])
        got = brute_lib.restricted_dp(x.ctypes.data_as(f32p), N, win.ctypes.data_as(f32p), win.shape[0], 1,
                                      0, hi - lo, a.ctypes.data_as(f32p), b.ctypes.data_as(f32p))
        assert np.float32(got) == c[q]


def test_deterministic_repeated_runs():
    """identical inputs give identical bits, run after run (persistent schedule,
    whose unit-to-worker assignment varies between runs)."""
    Q, Y = _inputs(300, 400, 60_000, 9)
    outs = [_gpu(Q, Y, trace=True) for _ in range(3)]
    for o in outs[1:]:
        for a, b in zip(outs[0], o):
            assert np.array_equal(np.asarray(a), np.asarray(b))


@pytest.mark.parametrize("fma", [1, 0])
def test_long_queries_single_row_layout(fma):
    """N = 8,000: the rows + boundary ring select the single-row query layout (one more
    resident CTA); bit-exact against the oracle like every other schedule."""
    Q, Y = _inputs(4, 8000, 20_000, 10)
    _check_exact(Q, Y, _gpu(Q, Y, OPT_FMA=fma), fma=bool(fma))


def test_cbf_inputs_bit_exact():
    """The paper's own test-data family (CBF)."""
    from datagen import cbf_batch, cbf_reference
    Y = oracle.znorm(cbf_reference(8000, 2)[None])[0]
    Q = oracle.znorm(cbf_batch(6, 256, 2))
    _check_exact(Q, Y, _gpu(Q, Y, trace=True), trace=True)


def test_max_size_reference_exact_match_at_the_far_end():
    """Maximum sizes: a 1.5e9-sample reference (6 GB, step and column counters near the int32
    limit of the kernel's planning) -- queries cut verbatim from the far end and from the start
    must score exactly 0 at their own end column (a property that holds at any size; raw mode),
    and a length past the ABI limit is rejected before anything is allocated."""
    M = 1_500_000_000
    rng = np.random.default_rng(77)
    Y = rng.standard_normal(M, dtype=np.float32)
    starts = [M - 64, M - 1_000_003, 12_345, 1_073_741_800]       # incl. one across 2^30
    Q = np.stack([Y[s:s + 64] for s in starts]).astype(np.float32)
    with sd.options(OPT_NORMALIZE=0):
        sd.set_reference(Y)
        del Y
        c, e = sd.batch(torch.as_tensor(Q, device=DEV))
    assert torch.all(c == 0).item(), c
    assert e.cpu().tolist() == [s + 63 for s in starts]
    sd.release()
    rc = sd._lib.sdtw_set_reference(ctypes.c_void_p(Q.ctypes.data), ctypes.c_int64(0x7fffffff))
    assert rc == sd.E_ARG


@pytest.mark.parametrize("fma", [1, 0])
@pytest.mark.parametrize("Z,N,M,opts", [
    (8, 64, 4096, dict()), (5, 300, 20001, dict()), (3, 1, 500, dict()), (4, 257, 3001, dict(OPT_LANES=2)),
    (6, 1000, 100_000, dict(OPT_SCHED=2, OPT_SEGMENTS=3)), (6, 1000, 100_000, dict(OPT_SCHED=3)),
    (6, 700, 50_000, dict(OPT_SCHED=1)),
])
def test_query_rows_in_global_memory(fma, Z, N, M, opts):
    """SDTW_OPT_QUERY_ROWS=2 (XG kernels: the query rows in a global pair-layout buffer instead
    of shared memory, the auto choice for long queries): bit-exact against the oracle for
    cost/end and the checkpointed start index, across schedules."""
    Q, Y = _inputs(Z, N, M, 90 + N)
    ref = oracle.sdtw(Q, Y, fma=bool(fma), start=True, last_rows=True)
    got = _gpu(Q, Y, OPT_FMA=fma, OPT_QUERY_ROWS=2, **opts)
    _check_exact(Q, Y, got, fma=bool(fma), ref=ref)
    if opts.get("OPT_SCHED") != 1:
        got_t = _gpu(Q, Y, trace=True, OPT_FMA=fma, OPT_QUERY_ROWS=2, OPT_START=2, **opts)
        _check_exact(Q, Y, got_t, fma=bool(fma), trace=True, ref=ref)
