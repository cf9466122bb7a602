"""GPU parity of the checkpointed start index (SDTW_OPT_START=2): the
cost/end DP stores every round's last column, then a window DP from the checkpoint left of
the end column and the paper's walk-back find the start.  It must give exactly the
forward-propagation start of reading G6 (OPT_START=1) and the oracle's, under every
schedule, including windows that must be widened (warp paths wider than a round) and
queries recomputed after a failed speculative correction; and sdtw_path's rows must equal
the oracle's walk-back."""
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


def _tb(Q, Y, **opts):
    kw = dict(OPT_NORMALIZE=0)
    kw.update(opts)
    with sd.options(**kw):
        sd.set_reference(torch.as_tensor(Y, device=DEV))
        c, e, s = sd.traceback(torch.as_tensor(np.ascontiguousarray(Q), device=DEV))
        fixed = sd.spec_recomputed()
    return c.cpu().numpy(), e.cpu().numpy(), s.cpu().numpy(), fixed


def _check(Q, Y, c, e, s, fma=True):
    ref = oracle.sdtw(Q, Y, fma=fma, start=True, last_rows=True)
    assert np.array_equal(c.view(np.uint32), ref["cost"].view(np.uint32)), (c[:4], ref["cost"][:4])
    assert np.array_equal(e, ref["end"]), (np.nonzero(e != ref["end"])[0][:8])
    assert np.array_equal(s, ref["start"]), (np.nonzero(s != ref["start"])[0][:8], s[:4], ref["start"][:4])


@pytest.mark.parametrize("fma", [1, 0])
@pytest.mark.parametrize("Z,N,M", [(8, 64, 4096), (5, 300, 20_001), (24, 500, 30_000), (6, 1000, 60_000),
                                   (3, 2000, 15_000), (7, 129, 4097)])
def test_ckpt_start_equals_forward_and_oracle(fma, Z, N, M):
    Q, Y = _inputs(Z, N, M, 100 + N)
    c2, e2, s2, _ = _tb(Q, Y, OPT_START=2, OPT_FMA=fma)
    c1, e1, s1, _ = _tb(Q, Y, OPT_START=1, OPT_FMA=fma)
    assert np.array_equal(c2, c1) and np.array_equal(e2, e1) and np.array_equal(s2, s1)
    _check(Q, Y, c2, e2, s2, fma=bool(fma))


@pytest.mark.parametrize("opts", [dict(OPT_SCHED=1), dict(OPT_SCHED=2, OPT_SEGMENTS=3), dict(OPT_SCHED=3),
                                  dict(OPT_LANES=1), dict(OPT_LANES=2, OPT_SCHED=3, OPT_SPEC_ROUNDS=1)])
def test_ckpt_start_all_schedules(opts):
    """One CTA per ring, sequential segments and speculative segments (whose checkpoints are
    merged with the corrections' inside the correction rounds) all give exact checkpoints."""
    Q, Y = _inputs(12, 400, 250_000, 77)
    c, e, s, _ = _tb(Q, Y, OPT_START=2, **opts)
    _check(Q, Y, c, e, s)


def test_ckpt_start_wide_paths_widen_the_window():
    """The reference holds 6 regions where each sample is repeated 6 times; the queries are
    the unstretched originals, so their cost-0 warp paths run ~3,000 columns wide: with
    one-warp rings (960 columns per round) the first window (2 rounds) is too narrow and the
    window must be widened, more than once for some."""
    base = oracle.znorm(nanopore_reference(60_000, 81)[None])[0]
    rng = np.random.default_rng(81)
    parts, Q = [], []
    pos = 0
    for a in sorted(rng.choice(np.arange(1000, 58_000, 9000), size=6, replace=False)):
        parts.append(base[pos:a])
        parts.append(np.repeat(base[a:a + 500], 6))
        Q.append(base[a:a + 500])
        pos = a + 500
    parts.append(base[pos:])
    Y = np.concatenate(parts).astype(np.float32)
    Q = np.stack(Q).astype(np.float32)
    c, e, s, _ = _tb(Q, Y, OPT_START=2, OPT_LANES=1)
    assert np.all(c == 0) and np.all(e - s > 2 * 960), (c, e - s)
    _check(Q, Y, c, e, s)


def test_ckpt_start_after_failed_corrections():
    """Reference copies across speculative segment boundaries with one-round corrections: the
    corrections are not overtaken, those queries are recomputed with one CTA per ring, and
    their checkpoints come from that recomputation."""
    M = 300_000
    Y = oracle.znorm(nanopore_reference(M, 83)[None])[0]
    Q0, _ = _inputs(4, 1500, M, 83)
    cpr, Sg = 960, 8                                  # one-warp rings: 32 x 2 chains x 15 columns
    Pr = -(-M // cpr)
    bounds = [(s * Pr // Sg) * cpr for s in (2, 4, 6)]   # segment boundaries (spec_table)
    cuts = [Y[b - 200:b + 1300] for b in bounds]      # copies running 1,300 columns past them
    Q = np.concatenate([np.stack(cuts), Q0]).astype(np.float32)
    c, e, s, fixed = _tb(Q, Y, OPT_START=2, OPT_SCHED=3, OPT_LANES=1, OPT_SPEC_ROUNDS=1, OPT_SEGMENTS=Sg)
    assert fixed >= 3
    assert np.all(c[:3] == 0) and np.array_equal(s[:3], np.array(bounds) - 200)
    _check(Q, Y, c, e, s)


def test_ckpt_start_ties():
    """Integer-valued inputs: exact ties everywhere; the priority rule decides the start."""
    rng = np.random.default_rng(85)
    Q = rng.integers(0, 3, (16, 40)).astype(np.float32)
    Y = rng.integers(0, 3, 9000).astype(np.float32)
    c, e, s, _ = _tb(Q, Y, OPT_START=2)
    _check(Q, Y, c, e, s)


def test_ckpt_path_equals_oracle_walkback():
    Q, Y = _inputs(4, 200, 12_000, 87)
    with sd.options(OPT_NORMALIZE=0, OPT_START=2):
        sd.set_reference(torch.as_tensor(Y, device=DEV))
        c, e, s, lo, hi = sd.path(torch.as_tensor(Q, device=DEV))
    c, e, s, lo, hi = [t.cpu().numpy() for t in (c, e, s, lo, hi)]
    for q in range(Q.shape[0]):
        rc, re, rs, rlo, rhi = oracle.sdtw_path(Q[q], Y)
        assert c[q] == rc and e[q] == re and s[q] == rs
        assert np.array_equal(lo[q], rlo) and np.array_equal(hi[q], rhi), q


def test_forced_ckpt_rejects_unqualified_launches():
    Q, Y = _inputs(2, 64, 4096, 89)
    with pytest.raises(sd.SdtwError) as ei:
        _tb(Q, Y, OPT_START=2, OPT_PACKED=0)
    assert ei.value.status == sd.E_ARG
    c, e, s, _ = _tb(Q, Y, OPT_START=0, OPT_PACKED=0)      # auto falls back to forward propagation
    _check(Q, Y, c, e, s)


def test_ckpt_start_two_segments():
    """Checkpointed start with the two-segment plan (first segment 16/25 of the rounds): the
    merge of the correction checkpoints uses the same split (spec_seg_start), both when the
    correction is overtaken (random queries, a copy straddling the midpoint) and when it fails
    (a copy straddling the split, recomputed)."""
    M = 200_000
    Y = oracle.znorm(nanopore_reference(M, 87)[None])[0]
    Q0, _ = _inputs(4, 1500, M, 87)
    cpr = 960
    Pr = -(-M // cpr)
    b = (Pr * 16 // 25) * cpr
    mid = (Pr // 2) * cpr
    Q = np.concatenate([np.stack([Y[b - 200:b + 1300], Y[mid - 200:mid + 1300]]), Q0]).astype(np.float32)
    c, e, s, fixed = _tb(Q, Y, OPT_START=2, OPT_SCHED=3, OPT_LANES=1, OPT_SPEC_ROUNDS=1, OPT_SEGMENTS=2)
    assert fixed >= 1
    assert c[0] == 0 and s[0] == b - 200 and c[1] == 0 and s[1] == mid - 200
    _check(Q, Y, c, e, s)
