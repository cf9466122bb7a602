"""GPU parity of the speculative-segment schedule (SDTW_OPT_SCHED=3): every
round-segment of a query starts at once from a +inf boundary, a correction pass of
OPT_SPEC_ROUNDS rounds per segment boundary repairs the result, and queries whose
correction is not overtaken in time are recomputed.  The result must be what the oracle
gives (cost bit-exact, end exact or a tie) and bit-identical to the sequential schedules,
both when the corrections succeed and when they are forced to fail, for cost / end and for
the start index."""
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


def _run(Q, Y, start=False, **opts):
    kw = dict(OPT_NORMALIZE=0)
    kw.update(opts)
    with sd.options(**kw):
        sd.set_reference(torch.as_tensor(Y, device=DEV))
        Qt = torch.as_tensor(np.ascontiguousarray(Q), device=DEV)
        out = sd.traceback(Qt) if start else sd.batch(Qt)
        torch.cuda.synchronize()
        fixed = sd.spec_recomputed()
        launches = sd.profile()[1]
    out = [o.cpu().numpy() for o in out]
    if start:
        return out[0], out[1], fixed, launches, out[2]
    return out[0], out[1], fixed, launches


def _check(Q, Y, c, e, fma=True, idx=None, s=None):
    idx = np.arange(len(Q)) if idx is None else np.asarray(idx)
    ref = oracle.sdtw(Q[idx], Y, fma=fma, last_rows=True, start=s is not None)
    assert np.array_equal(c[idx].view(np.uint32), ref["cost"].view(np.uint32)), (c[idx][:4], ref["cost"][:4])
    for k in np.nonzero(e[idx] != ref["end"])[0]:
        assert ref["last_rows"][k, e[idx][k]] == ref["cost"][k], (k, e[idx][k], ref["end"][k])
    if s is not None:
        same = e[idx] == ref["end"]
        assert np.array_equal(s[idx][same], ref["start"][same]), (s[idx][:4], ref["start"][:4])


@pytest.mark.parametrize("fma", [1, 0])
def test_spec_small_bit_exact(fma):
    Q, Y = _inputs(6, 300, 200_000, 61)
    c, e, fixed, _ = _run(Q, Y, OPT_SCHED=3, OPT_FMA=fma)
    _check(Q, Y, c, e, bool(fma))


@pytest.mark.parametrize("fma", [1, 0])
def test_spec_start_index_bit_exact(fma):
    Q, Y = _inputs(6, 300, 200_000, 66)
    c, e, fixed, _, s = _run(Q, Y, start=True, OPT_SCHED=3, OPT_FMA=fma)
    _check(Q, Y, c, e, bool(fma), s=s)
    a = _run(Q, Y, start=True, OPT_SCHED=1, OPT_FMA=fma)
    assert np.array_equal(c.view(np.uint32), a[0].view(np.uint32))
    assert np.array_equal(e, a[1]) and np.array_equal(s, a[4])


def test_spec_start_index_embedded_matches():
    """Exact embeddings (cost 0, known start / end) spread over the reference, some across
    segment boundaries: start columns exact."""
    M, N = 300_000, 400
    Y = oracle.znorm(nanopore_reference(M, 67)[None])[0]
    rng = np.random.default_rng(67)
    starts = np.sort(rng.integers(0, M - N, 10))
    Q = np.stack([Y[a:a + N] for a in starts]).astype(np.float32)
    c, e, fixed, _, s = _run(Q, Y, start=True, OPT_SCHED=3, OPT_SEGMENTS=20)
    assert np.all(c == 0) and np.array_equal(s, starts) and np.array_equal(e, starts + N - 1)


def test_spec_matches_sequential_schedules():
    Q, Y = _inputs(20, 2000, 1_000_000, 62)
    a = _run(Q, Y, OPT_SCHED=1)
    b = _run(Q, Y, OPT_SCHED=3)
    c = _run(Q, Y)                                  # auto: small batch -> speculative
    for got in (b, c):
        assert np.array_equal(got[0].view(np.uint32), a[0].view(np.uint32)) and np.array_equal(got[1], a[1])
    assert c[3] == 3                                # normalise-check, DP, speculative finalize
    _check(Q, Y, b[0], b[1], idx=[0, 7, 19])


def test_spec_forced_recompute_is_exact():
    """Queries that are exact copies of the reference across a segment boundary: the path
    entering from the boundary scores ~0 for longer than a one-round correction (one-warp
    rings: 960 columns per round), so the corrections fail and the queries are recomputed."""
    M, N, Sg = 100_000, 1500, 8
    Y = oracle.znorm(nanopore_reference(M, 63)[None])[0]
    Pr = -(-M // 960)
    bounds = [(s * Pr // Sg) * 960 for s in range(1, 6)]
    Q = np.stack([Y[b - 200:b + N - 200] for b in bounds]).astype(np.float32)
    c, e, fixed, _ = _run(Q, Y, OPT_SCHED=3, OPT_LANES=1, OPT_SPEC_ROUNDS=1, OPT_SEGMENTS=Sg)
    assert fixed == len(bounds)
    _check(Q, Y, c, e)
    assert np.all(c == 0) and np.array_equal(e, np.array(bounds) + N - 201)
    c, e, fixed, _, st = _run(Q, Y, start=True, OPT_SCHED=3, OPT_LANES=1, OPT_SPEC_ROUNDS=1, OPT_SEGMENTS=Sg)
    assert fixed == len(bounds) and np.all(c == 0) and np.array_equal(st, np.array(bounds) - 200)


def test_spec_ragged_forced_recompute_is_exact():
    """Ragged batch: reads copying the reference across segment boundaries (recomputed through
    a ragged sub-batch) next to random reads (not recomputed); every result exact."""
    M, Sg = 100_000, 8
    Y = oracle.znorm(nanopore_reference(M, 68)[None])[0]
    Pr = -(-M // 960)
    bounds = [(s * Pr // Sg) * 960 for s in (1, 3, 5)]
    lens = [1500, 1300, 1700]
    qs = [Y[b - 200:b - 200 + n].astype(np.float32) for b, n in zip(bounds, lens)]
    qs += [oracle.znorm(nanopore_queries(1, n, M, 680 + n))[0] for n in (90, 400, 1100)]
    off = np.zeros(len(qs) + 1, np.int64)
    off[1:] = np.cumsum([len(q) for q in qs])
    with sd.options(OPT_NORMALIZE=0, OPT_SCHED=3, OPT_LANES=1, OPT_SPEC_ROUNDS=1, OPT_SEGMENTS=Sg):
        sd.set_reference(Y)
        c, e, st = sd.batch_ragged(np.concatenate(qs), off, start=True)
        fixed = sd.spec_recomputed()
    assert fixed >= 3
    for k, q in enumerate(qs):
        r = oracle.sdtw(q[None], Y, start=True, last_rows=True)
        assert c[k] == r["cost"][0], k
        if e[k] != r["end"][0]:
            assert r["last_rows"][0, e[k]] == r["cost"][0], k
        else:
            assert st[k] == r["start"][0], k
    assert np.all(c[:3] == 0) and np.array_equal(st[:3], np.array(bounds) - 200)


def test_spec_short_corrections_mixed():
    """Corrections of one round on a short query: most succeed; exact either way."""
    Q, Y = _inputs(12, 120, 300_000, 64)
    c, e, fixed, _ = _run(Q, Y, OPT_SCHED=3, OPT_SPEC_ROUNDS=1, OPT_SEGMENTS=20)
    assert fixed < 12
    _check(Q, Y, c, e)
    a = _run(Q, Y, OPT_SCHED=1)
    assert np.array_equal(c.view(np.uint32), a[0].view(np.uint32)) and np.array_equal(e, a[1])


def test_spec_constant_signals_ties():
    """All-zero inputs: every cell is 0, the boundary DP ties the free DP everywhere; the
    end is the smallest column of the last row (N-1)."""
    Y = np.zeros(150_000, np.float32)
    Q = np.zeros((3, 200), np.float32)
    c, e, fixed, _ = _run(Q, Y, OPT_SCHED=3)
    assert np.all(c == 0) and np.all(e == 0) and fixed == 0
    # start index by forward propagation: the tie between boundary and free paths is not a
    # strict win -> recompute
    c, e, fixed, _, s = _run(Q, Y, start=True, OPT_SCHED=3, OPT_START=1)
    assert np.all(c == 0) and np.all(e == 0) and np.all(s == 0) and fixed == 3
    # checkpointed start index: the cost/end DP's values are exact under ties
    # (min of the two DPs), and the start comes from the walk-back on them -- no recompute
    c, e, fixed, _, s = _run(Q, Y, start=True, OPT_SCHED=3, OPT_START=2)
    assert np.all(c == 0) and np.all(e == 0) and np.all(s == 0) and fixed == 0


def test_spec_errors():
    Q, Y = _inputs(2, 50, 100_000, 65)
    with sd.options(OPT_NORMALIZE=0, OPT_SCHED=3):
        sd.set_reference(Y)
        with sd.options(OPT_CLUSTER=2):
            with pytest.raises(sd.SdtwError):
                sd.batch(Q)                          # one CTA per ring only
        bad = Q.copy()
        bad[1, 3] = np.nan
        with pytest.raises(sd.SdtwError) as ei:
            sd.batch(bad)
        assert ei.value.status == sd.E_NONFINITE


@pytest.mark.parametrize("Z,N,M,start", [(1, 2000, 10_000_000, False), (1, 500, 2_000_000, True),
                                         (2048, 300, 1_000_000, False), (3, 8000, 3_000_000, False),
                                         (700, 64, 500_000, True)])
def test_spec_edge_shapes_identical_to_sequential(Z, N, M, start):
    """One query (hundreds of segments), thousands of queries (two segments), single-row
    layout (N=8,000), short queries with start index: bit-identical to sequential segments."""
    Y = torch.from_numpy(nanopore_reference(M, 5)).to(DEV)
    Q = torch.from_numpy(nanopore_queries(Z, N, M, 5)).to(DEV)
    sd.set_reference(Y)
    run = sd.traceback if start else sd.batch
    with sd.options(OPT_SCHED=3):
        a = [t.cpu() for t in run(Q)]
    with sd.options(OPT_SCHED=2):
        b = [t.cpu() for t in run(Q)]
    assert all(torch.equal(x, y) for x, y in zip(a, b))


def test_nested_recomputation_levels_are_exact():
    """Failed queries are re-run as their own speculative batch with corrections x4 (DESIGN.md
    §13); on a fully 5x-oversampled reference with one-round corrections some of THOSE fail
    again (a second level, OPT_STAT_FIXUP_DEPTH = 2), each level in its own workspace --
    cost, end and (checkpointed) start all exact against the oracle."""
    import oracle
    from datagen import nanopore_reference
    M, N, Z, seed = 100_000, 1500, 12, 81
    levels = oracle.znorm(nanopore_reference(M // 5 + 10, seed)[None])[0]
    Y = np.repeat(levels, 5)[:M].astype(np.float32)
    rng = np.random.default_rng(seed)
    starts = rng.integers(0, M // 5 - N - 1, size=Z)
    Q = np.stack([levels[s:s + N] + 0.05 * rng.standard_normal(N) for s in starts]).astype(np.float32)
    ref = oracle.sdtw(Q, Y, start=True)
    with sd.options(OPT_NORMALIZE=0, OPT_SCHED=3, OPT_LANES=1, OPT_SPEC_ROUNDS=1):
        sd.set_reference(torch.as_tensor(Y, device="cuda"))
        c, e = sd.batch(torch.as_tensor(Q, device="cuda"))
        assert sd.spec_recomputed() == Z and sd.get_option(sd.OPT_STAT_FIXUP_DEPTH) >= 2
        c2, e2, s2 = sd.traceback(torch.as_tensor(Q, device="cuda"))
    for cc, ee in ((c, e), (c2, e2)):
        assert np.array_equal(cc.cpu().numpy().view(np.uint32), ref["cost"].view(np.uint32))
        assert np.array_equal(ee.cpu().numpy(), ref["end"])
    assert np.array_equal(s2.cpu().numpy(), ref["start"])


def test_spec_two_segments_split_point():
    """The two-segment plan splits at 16/25 of the rounds (spec_seg_start):
    queries copying the reference across THAT boundary defeat one-round corrections and are
    recomputed (so may others: with N = 1,500 rows against a 960-column correction any query's
    correction can fail -- the auto correction covers N columns plus half a round); a copy straddling the
    midpoint, random queries; every result exact against the oracle and the sequential schedule."""
    M, N = 100_000, 1500
    Y = oracle.znorm(nanopore_reference(M, 64)[None])[0]
    Pr = -(-M // 960)                               # one-warp rings: 960 columns per round
    b = (Pr * 16 // 25) * 960                       # the split column
    mid = (Pr // 2) * 960
    Q0, _ = _inputs(3, N, M, 64)
    Q = np.concatenate([np.stack([Y[b - 200:b + N - 200], Y[mid - 200:mid + N - 200]]), Q0]).astype(np.float32)
    c, e, fixed, _ = _run(Q, Y, OPT_SCHED=3, OPT_LANES=1, OPT_SPEC_ROUNDS=1, OPT_SEGMENTS=2)
    assert fixed >= 1
    _check(Q, Y, c, e)
    assert c[0] == 0 and e[0] == b + N - 201 and c[1] == 0 and e[1] == mid + N - 201
    _, _, fixed2, _ = _run(Q[:1], Y, OPT_SCHED=3, OPT_LANES=1, OPT_SPEC_ROUNDS=1, OPT_SEGMENTS=2)
    assert fixed2 == 1                              # the copy across the split defeats its correction
    cs, es, _, _ = _run(Q, Y, OPT_SCHED=2, OPT_LANES=1, OPT_SEGMENTS=2)
    assert np.array_equal(c.view(np.uint32), cs.view(np.uint32)) and np.array_equal(e, es)
    c, e, fixed, _, st = _run(Q, Y, start=True, OPT_SCHED=3, OPT_LANES=1, OPT_SPEC_ROUNDS=1, OPT_SEGMENTS=2)
    assert fixed >= 1 and st[0] == b - 200 and st[1] == mid - 200
    _check(Q, Y, c, e, s=st)
