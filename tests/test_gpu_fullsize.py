"""Full-size GPU parity: the exact launches bench.py times, checked
against the CPU oracle on the WHOLE reference for a deterministic query subset.

* config 3 (the headline: 512 x 2,000 vs 10M, z-normalisation inside the call, default
  speculative schedule): every 32nd query against `oracle.sdtw(znorm(Q), znorm(Y))` on the
  full 10M reference -- cost BIT-EXACT (both normalisers use exact sums, G8), end
  exact or a tie in the oracle's last row (G5).
* config 5 N = 4,000 / 8,000 with the start index (512 queries vs 1M): a query subset
  against the full-reference oracle -- cost bit-exact, end exact or tied, start exact when
  the end is the oracle's, and in every case VALID: a DP restricted to begin exactly at the
  GPU's start column reproduces the cost at the GPU's end column (SURVEY §8(c) agreement 4).

The oracle runs on the host cores (16 threads on the B200 box: ~150 s for config 3, about
60 s for config 5).  PAPER.md P:L124 (correctness against the CPU sequential output) on the
paper's batch."""
import ctypes
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle  # noqa: E402
import paper_2403_06931_b200 as sd  # noqa: E402
from datagen import CONFIGS, nanopore_queries, nanopore_reference  # noqa: E402

DEV = torch.device("cuda", 0)
f32p = ctypes.POINTER(ctypes.c_float)


def _restricted(brute_lib, x, Y, start, end):
    """D(N-1, end) of the DP that may only begin at column `start` (window [start, end])."""
    win = np.ascontiguousarray(Y[start:end + 1])
    x = np.ascontiguousarray(x, np.float32)
    a = np.empty(win.shape[0], np.float32)
    b = np.empty(win.shape[0], np.float32)
    return np.float32(brute_lib.restricted_dp(x.ctypes.data_as(f32p), x.shape[0], win.ctypes.data_as(f32p),
                                              win.shape[0], 1, 0, end - start, a.ctypes.data_as(f32p),
                                              b.ctypes.data_as(f32p)))


def _tie_ok(xn, Yn, end_gpu, cost):
    """The oracle's last-row value at the GPU's end column equals the minimum (a tie)."""
    r = oracle.sdtw(xn[None], Yn, last_rows=True)
    return r["last_rows"][0, end_gpu] == cost


def _bench_launch(name, trace):
    """The bench's own call: raw inputs, library normalisation on, default options."""
    cfg = CONFIGS[name]
    Y = nanopore_reference(cfg["M"], cfg["seed"])
    Q = nanopore_queries(cfg["Z"], cfg["N"], cfg["M"], cfg["seed"])
    sd.set_reference(torch.as_tensor(Y, device=DEV))
    Qd = torch.as_tensor(Q, device=DEV)
    out = sd.traceback(Qd) if trace else sd.batch(Qd)
    return Q, Y, [o.cpu().numpy() for o in out]


def test_config3_headline_vs_full_reference_oracle():
    Q, Y, (c, e) = _bench_launch("c3", trace=False)
    assert sd.spec_recomputed() >= 0
    idx = np.arange(0, Q.shape[0], 32)                       # 16 queries, every rank-8 shard covered
    Yn = oracle.znorm(Y[None])[0]
    Qn = oracle.znorm(Q[idx])
    ref = oracle.sdtw(Qn, Yn)
    assert np.array_equal(c[idx].view(np.uint32), ref["cost"].view(np.uint32)), \
        (idx[c[idx] != ref["cost"]], c[idx][:4], ref["cost"][:4])
    for k in np.nonzero(e[idx] != ref["end"])[0]:
        assert _tie_ok(Qn[k], Yn, e[idx][k], ref["cost"][k]), (idx[k], e[idx][k], ref["end"][k])


@pytest.mark.parametrize("name,step", [("c5_500", 16), ("c5_1000", 16), ("c5_4000", 32), ("c5_8000", 64)])
def test_config5_start_index_vs_full_reference_oracle(brute_lib, name, step):
    Q, Y, (c, e, s) = _bench_launch(name, trace=True)
    idx = np.arange(0, Q.shape[0], step)
    Yn = oracle.znorm(Y[None])[0]
    Qn = oracle.znorm(Q[idx])
    ref = oracle.sdtw(Qn, Yn, start=True)
    assert np.array_equal(c[idx].view(np.uint32), ref["cost"].view(np.uint32))
    for k, q in enumerate(idx):
        if e[q] == ref["end"][k]:
            assert s[q] == ref["start"][k], (q, s[q], ref["start"][k])
        else:
            assert _tie_ok(Qn[k], Yn, e[q], ref["cost"][k]), (q, e[q], ref["end"][k])
        assert 0 <= s[q] <= e[q]
        assert _restricted(brute_lib, Qn[k], Yn, int(s[q]), int(e[q])) == c[q], q


def test_config4_batch_on_one_gpu_vs_full_reference_oracle():
    """Config 4's batch (4,096 x 2,000 vs 10M; 512 per GPU at 8 GPUs) in ONE launch on the
    test GPU: 4 queries (one per two 512-query rank shards) against the full-reference oracle."""
    Q, Y, (c, e) = _bench_launch("c4", trace=False)
    idx = np.arange(0, Q.shape[0], 1024) + 37                # 4 queries, one per pair of rank shards
    Yn = oracle.znorm(Y[None])[0]
    Qn = oracle.znorm(Q[idx])
    ref = oracle.sdtw(Qn, Yn)
    assert np.array_equal(c[idx].view(np.uint32), ref["cost"].view(np.uint32))
    for k in np.nonzero(e[idx] != ref["end"])[0]:
        assert _tie_ok(Qn[k], Yn, e[idx][k], ref["cost"][k])


def test_config3_straddle_worst_case_vs_full_reference_oracle():
    """The speculative schedule's adversarial workload (bench c3_straddle):
    64 queries whose paths overrun the correction pass are recomputed (as their own
    speculative batch); 4 of them and 2 benign queries against the full-reference oracle."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("_bench", os.path.join(os.path.dirname(os.path.dirname(
        os.path.abspath(__file__))), "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    with sd.options(OPT_SEGMENTS=6):
        Q, Y, w = bench._workload("c3_straddle", 0, 1, "strong")
        sd.set_reference(torch.as_tensor(Y, device=DEV))
        c, e = [o.cpu().numpy() for o in sd.batch(torch.as_tensor(Q, device=DEV))]
        assert sd.spec_recomputed() == 64
    idx = np.array([0, 136, 256, 504, 1, 301])               # 4 straddling queries, 2 benign
    Yn = oracle.znorm(Y[None])[0]
    Qn = oracle.znorm(Q[idx])
    ref = oracle.sdtw(Qn, Yn)
    assert np.array_equal(c[idx].view(np.uint32), ref["cost"].view(np.uint32))
    for k in np.nonzero(e[idx] != ref["end"])[0]:
        assert _tie_ok(Qn[k], Yn, e[idx][k], ref["cost"][k])
