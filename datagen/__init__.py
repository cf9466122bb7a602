"""Seeded synthetic inputs for the sDTW hot path.

This module holds NONE of the method's arithmetic (no distance, no recurrence,
no normalisation): it only draws seeded random series with the shapes and value
distributions of the paper's workloads. Both the oracle tests and the CUDA path
are fed from here; neither side imports the other.

Two families (recipe stated in DESIGN.md §3):

* ``nanopore`` (primary, BASELINE.json "synthetic nanopore-like signals"):
  a random genome over {A,C,G,T}, a 6-mer level table ~ N(0,1), the reference is
  one level per base; a query is a genome window (50 % cut from the reference
  genome, 50 % from an independent genome), each base held 1+Poisson(8)
  samples, Gaussian noise sigma=0.2, a random affine map, then mapped to a raw
  pA-like scale (90 + 12*s) and truncated to N samples.
* ``cbf`` (the paper's own generator family, §4
  "make_cylinder_bell_funnel"; construction as SPEC.md S:L397-L445).

Seeds per config follow SURVEY.md §8(d): C1=1, C2=2, C3=3, C4=4, C5=5.
"""
from __future__ import annotations

import numpy as np

__all__ = [
    "CONFIGS",
    "nanopore_reference",
    "nanopore_queries",
    "nanopore_workload",
    "nanopore_ragged",
    "cbf_series",
    "cbf_reference",
    "cbf_batch",
    "embed_queries",
    "straddle_workload",
]

# name -> (Z, N, M, seed, traceback)
CONFIGS = {
    "c1": dict(Z=8, N=64, M=4096, seed=1, start=False),
    "c2": dict(Z=512, N=2000, M=100_000, seed=2, start=False),
    "c3": dict(Z=512, N=2000, M=10_000_000, seed=3, start=False),
    "c4": dict(Z=4096, N=2000, M=10_000_000, seed=4, start=False),
    "c5_500": dict(Z=512, N=500, M=1_000_000, seed=5, start=True),
    "c5_1000": dict(Z=512, N=1000, M=1_000_000, seed=5, start=True),
    "c5_4000": dict(Z=512, N=4000, M=1_000_000, seed=5, start=True),
    "c5_8000": dict(Z=512, N=8000, M=1_000_000, seed=5, start=True),
    # the paper's generator family (CBF) at config-2 shape: throughput is data-oblivious
    "c2_cbf": dict(Z=512, N=2000, M=100_000, seed=2, start=False, cbf=True),
    # config 3 with 1/8 of the queries matching oversampled reference regions that straddle
    # the speculative segment boundaries (the schedule's worst case)
    "c3_straddle": dict(Z=512, N=2000, M=10_000_000, seed=3, start=False, straddle=(8, 5)),
    # NEXT-4: a ragged batch of reads, lengths log-uniform in [500, 8000] (N = mean, info only)
    "c6_ragged": dict(Z=512, N=2700, M=1_000_000, seed=6, start=False, ragged=(500, 8000)),
}

_K = 6  # k-mer order of the level table


def _rng(seed: int, stream: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64([int(seed), int(stream)]))


def _levels(seed: int) -> np.ndarray:
    return _rng(seed, 0).standard_normal(4 ** _K)


def _genome(rng: np.random.Generator, n_bases: int) -> np.ndarray:
    return rng.integers(0, 4, size=n_bases, dtype=np.int64)


def _kmer_signal(genome: np.ndarray, levels: np.ndarray) -> np.ndarray:
    """One expected level per base: level of the 6-mer starting at that base."""
    n = genome.shape[0] - _K + 1
    idx = np.zeros(n, dtype=np.int64)
    for k in range(_K):
        idx = idx * 4 + genome[k:k + n]
    return levels[idx]


def _ref_genome(seed: int, M: int) -> np.ndarray:
    return _genome(_rng(seed, 1), M + _K - 1)


def nanopore_reference(M: int, seed: int) -> np.ndarray:
    """Reference = pore-model expected signal, one sample per base, M samples (fp32)."""
    return _kmer_signal(_ref_genome(seed, M), _levels(seed)).astype(np.float32)


def nanopore_queries(Z: int, N: int, M: int, seed: int,
                     on_target: float = 0.5, first_query: int = 0) -> np.ndarray:
    """Z x N raw (pA-like) queries, row-major, contiguous (§5.1).

    Queries first_query .. first_query+Z-1 of the stream for (seed, M): a rank of a
    sharded job generates only its own shard."""
    levels = _levels(seed)
    ref_genome = _ref_genome(seed, M)
    out = np.empty((Z, N), dtype=np.float32)
    for q in range(Z):
        rng = _rng(seed, 1000 + first_query + q)
        n_bases = max(8, N // 9 + 16)
        while True:
            if rng.random() < on_target and M >= n_bases + _K:
                off = int(rng.integers(0, M - n_bases + 1))
                g = ref_genome[off:off + n_bases + _K - 1]
            else:
                g = _genome(rng, n_bases + _K - 1)
            sig = _kmer_signal(g, levels)
            dwell = 1 + rng.poisson(8.0, size=sig.shape[0])
            s = np.repeat(sig, dwell)
            if s.shape[0] >= N:
                break
            n_bases *= 2
        s = s[:N] + 0.2 * rng.standard_normal(N)
        scale = rng.uniform(0.8, 1.25)
        offset = 0.5 * rng.standard_normal()
        out[q] = (90.0 + 12.0 * (scale * s + offset)).astype(np.float32)
    return out


def nanopore_ragged(Z: int, M: int, seed: int, lmin: int, lmax: int, first_query: int = 0):
    """Variable-length reads (read-until style): lengths log-uniform in
    [lmin, lmax], each read generated as nanopore_queries would.  Returns (Q concatenated
    fp32, offsets int64 [Z+1])."""
    lens = np.empty(Z, np.int64)
    for q in range(Z):
        rng = _rng(seed, 500_000 + first_query + q)
        lens[q] = int(np.exp(rng.uniform(np.log(lmin), np.log(lmax))))
    parts = [nanopore_queries(1, int(lens[q]), M, seed, first_query=first_query + q)[0] for q in range(Z)]
    off = np.zeros(Z + 1, np.int64)
    off[1:] = np.cumsum(lens)
    return np.concatenate(parts).astype(np.float32), off


def nanopore_workload(name: str):
    """(Q[Z,N] fp32, Y[M] fp32, cfg) for a named config of BASELINE.json."""
    cfg = CONFIGS[name]
    Y = nanopore_reference(cfg["M"], cfg["seed"])
    Q = nanopore_queries(cfg["Z"], cfg["N"], cfg["M"], cfg["seed"])
    return Q, Y, cfg


# --- CBF, the paper's generator family ---

def cbf_series(length: int, rng: np.random.Generator, shape: int | None = None) -> np.ndarray:
    if length < 16:
        raise ValueError("cbf length must be >= 16")
    if shape is None:
        shape = int(rng.integers(0, 3))
    a = int(rng.integers(-(-length // 8), -(-length // 4) + 1))
    dur = int(rng.integers(-(-length // 4), -(-3 * length // 4) + 1))
    b = min(a + dur, length)
    amp = 6.0 + rng.standard_normal()
    t = np.arange(length, dtype=np.float64)
    inside = (t >= a) & (t <= b)
    if shape == 0:      # cylinder
        env = inside.astype(np.float64)
    elif shape == 1:    # bell
        env = np.where(inside, (t - a) / max(b - a, 1), 0.0)
    else:               # funnel
        env = np.where(inside, (b - t) / max(b - a, 1), 0.0)
    return amp * env + rng.standard_normal(length)


def cbf_reference(M: int, seed: int) -> np.ndarray:
    rng = _rng(seed, 2)
    n_win = -(-M // 128)
    return np.concatenate([cbf_series(128, rng) for _ in range(n_win)])[:M].astype(np.float32)


def cbf_batch(Z: int, N: int, seed: int) -> np.ndarray:
    out = np.empty((Z, N), dtype=np.float32)
    for q in range(Z):
        rng = _rng(seed, 5000 + q)
        n_win = -(-N // 128)
        out[q] = np.concatenate([cbf_series(128, rng) for _ in range(n_win)])[:N]
    return out


def embed_queries(Y: np.ndarray, Z: int, N: int, seed: int, stretch: int = 1):
    """Queries cut verbatim from Y (optionally each sample repeated `stretch` times).

    Returns (Q[Z, N*stretch], starts[Z]). Used for the embedding / time-stretch
    invariants (BASELINE.json "Oracle" invariants)."""
    rng = _rng(seed, 7)
    M = Y.shape[0]
    starts = rng.integers(0, M - N + 1, size=Z)
    Q = np.stack([np.repeat(Y[s:s + N], stretch) for s in starts]).astype(np.float32)
    return Q, starts.astype(np.int64)


def straddle_workload(Y: np.ndarray, boundaries, Z_per: int, N: int, stride: int, lead: int, seed: int):
    """The speculative schedule's adversarial case: around each boundary b
    the reference is replaced on [b - lead, b - lead + N*stride) by a `stride`x oversampled
    level sequence L (each of N levels held `stride` samples, as in a slow-translocation /
    repeat region), and Z_per queries per boundary are L plus Gaussian noise (0.2 level
    units).  Their optimal paths start before b and run N*stride - lead columns past it.
    Returns (Y', Q[len(boundaries)*Z_per, N])."""
    rng = _rng(seed, 9)
    Y = np.array(Y, dtype=np.float32, copy=True)
    qs = []
    for b in boundaries:
        p = int(b) - lead
        L = Y[p:p + N].copy()
        Y[p:p + N * stride] = np.repeat(L, stride)
        for _ in range(Z_per):
            qs.append(L + 0.2 * rng.standard_normal(N))
    return Y, np.stack(qs).astype(np.float32)
