"""GPU parity of sdtw_batch_ragged (batches of variable-length reads).

Every query of a ragged batch must give exactly what the oracle gives for that query
alone (raw mode, same FMA mode: cost bit-exact, end / start exact or a tie), and a
ragged batch of equal lengths must be bit-identical to the fixed-length batch.
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


def _ragged_inputs(lengths, M, seed):
    Y = oracle.znorm(nanopore_reference(M, seed)[None])[0]
    rng = np.random.default_rng(seed)
    qs = [oracle.znorm(nanopore_queries(1, int(n), M, seed + 17 * k)) [0] for k, n in enumerate(lengths)]
    off = np.zeros(len(lengths) + 1, np.int64)
    off[1:] = np.cumsum(lengths)
    del rng
    return qs, np.concatenate(qs).astype(np.float32), off, Y


def _check(qs, Y, c, e, s, fma, idx=None):
    for q in (range(len(qs)) if idx is None else idx):
        r = oracle.sdtw(qs[q][None], Y, fma=fma, start=s is not None, last_rows=True)
        assert c[q].view(np.uint32) == r["cost"][0].view(np.uint32), (q, c[q], r["cost"][0])
        if e[q] != r["end"][0]:
            assert r["last_rows"][0, e[q]] == r["cost"][0], q
        elif s is not None:
            assert s[q] == r["start"][0], q


@pytest.mark.parametrize("fma", [1, 0])
@pytest.mark.parametrize("start", [False, True])
def test_ragged_small_bit_exact(fma, start):
    rng = np.random.default_rng(3 + fma)
    lengths = rng.integers(1, 700, 20)
    lengths[0], lengths[1] = 1, 64
    qs, Q, off, Y = _ragged_inputs(lengths, 4096, 21)
    with sd.options(OPT_NORMALIZE=0, OPT_FMA=fma):
        sd.set_reference(torch.as_tensor(Y, device=DEV))
        out = sd.batch_ragged(torch.as_tensor(Q, device=DEV), torch.as_tensor(off, device=DEV), start=start)
    c, e = out[0].cpu().numpy(), out[1].cpu().numpy()
    s = out[2].cpu().numpy() if start else None
    _check(qs, Y, c, e, s, bool(fma))


def test_ragged_equal_lengths_match_fixed_batch():
    """Persistent schedule (Z > #SMs): equal lengths give the fixed-length results bit for bit."""
    Z, N, M = 300, 500, 100_000
    Y = oracle.znorm(nanopore_reference(M, 4)[None])[0]
    Q = oracle.znorm(nanopore_queries(Z, N, M, 4))
    off = np.arange(Z + 1, dtype=np.int64) * N
    with sd.options(OPT_NORMALIZE=0):
        sd.set_reference(torch.as_tensor(Y, device=DEV))
        Qt = torch.as_tensor(Q, device=DEV)
        c0, e0, s0 = sd.traceback(Qt)
        c1, e1, s1 = sd.batch_ragged(Qt.reshape(-1), off, start=True)
    assert torch.equal(c0, c1) and torch.equal(e0, e1) and torch.equal(s0, s1)


def test_ragged_persistent_mixed_lengths_sampled():
    rng = np.random.default_rng(8)
    lengths = np.exp(rng.uniform(np.log(200), np.log(1500), 300)).astype(np.int64)
    qs, Q, off, Y = _ragged_inputs(lengths, 60_000, 8)
    with sd.options(OPT_NORMALIZE=0):
        sd.set_reference(Y)
        c, e, s = sd.batch_ragged(Q, off, start=True)
    idx = list(rng.choice(300, 10, replace=False)) + [int(np.argmax(lengths)), int(np.argmin(lengths))]
    _check(qs, Y, c, e, s, True, idx)


def test_ragged_normalised_end_to_end():
    """With normalisation on, each query is z-normalised with its own statistics."""
    rng = np.random.default_rng(5)
    lengths = rng.integers(50, 400, 12)
    Yraw = nanopore_reference(5000, 5)
    raw = [nanopore_queries(1, int(n), 5000, 50 + k)[0] for k, n in enumerate(lengths)]
    off = np.zeros(13, np.int64)
    off[1:] = np.cumsum(lengths)
    sd.set_reference(Yraw)
    c, e = sd.batch_ragged(np.concatenate(raw).astype(np.float32), off)
    Yn = oracle.znorm(Yraw[None])[0]
    for q in range(12):
        r = oracle.sdtw(oracle.znorm(raw[q][None]), Yn, last_rows=True)
        assert abs(float(c[q]) - float(r["cost"][0])) <= 1e-5 * max(1.0, float(r["cost"][0])), q


def test_ragged_errors_and_empty():
    with sd.options(OPT_NORMALIZE=0):
        sd.set_reference(np.zeros(100, np.float32))
        for bad in ([1, 5], [0, 0, 3], [0, 4, 2]):
            with pytest.raises(sd.SdtwError) as e:
                sd.batch_ragged(np.zeros(8, np.float32), np.array(bad, np.int64))
            assert e.value.status == sd.E_ARG
        c, e = sd.batch_ragged(np.zeros(0, np.float32), np.zeros(1, np.int64))
        assert c.shape == (0,)


def test_ragged_long_reads_bit_exact():
    """Reads up to 9,000 samples (single-row query layout) next to short ones."""
    lengths = np.array([9000, 120, 4000, 700, 8800, 33])
    qs, Q, off, Y = _ragged_inputs(lengths, 15_000, 12)
    with sd.options(OPT_NORMALIZE=0):
        sd.set_reference(Y)
        c, e = sd.batch_ragged(Q, off)
    _check(qs, Y, c, e, None, True)
