/*
 * sdtw.h -- C ABI of the B200-native batched subsequence-DTW engine
 * (arXiv 2403.06931, "sDTW on AMD GPUs with HIP/ROCm"; citations P:Lnn are
 * lines of that paper's PAPER.md, S:Lnn of SPEC.md).
 *
 * Problem (§2, Eq. 1): for every query X (length N) of a
 * batch, fill the N x M matrix
 *     D(i,j) = min{D(i-1,j), D(i,j-1), D(i-1,j-1)} + (X_i - Y_j)^2
 * against one long reference Y (length M), with a free start anywhere in row 0
 * (virtual row -1 = 0, virtual column -1 = +inf), and report
 *     cost = min_j D(N-1,j),  end = smallest j attaining it,
 * and optionally the start column of that warp path (P:L35 walk-back).
 * Everything is fp32; see DESIGN.md §2 for every reading of the paper.
 *
 * Threading / devices: one library context per CUDA device; every call acts on
 * the CURRENT device (cudaGetDevice).  A multi-GPU job runs one process per
 * GPU and calls the ABI once per rank.  Calls are not re-entrant on one device.
 *
 * Pointers: Q / in / out / Y may be host or device pointers (detected with
 * cudaPointerGetAttributes; device pointers must live on the current device).
 * The caller owns them.  All calls are synchronous: they return after the
 * results are written (work is enqueued on the SDTW_OPT_STREAM stream, then
 * that stream is synchronised).  No partial results are written on error.
 */
#ifndef SDTW_H
#define SDTW_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    SDTW_OK = 0,
    SDTW_E_ARG = 1,        /* N<1, M<1, n<0, NULL pointer with n>0, bad option */
    SDTW_E_NOREF = 2,      /* sdtw_batch/traceback before sdtw_set_reference */
    SDTW_E_CUDA = 3,       /* CUDA runtime error (text in sdtw_last_error) */
    SDTW_E_NOMEM = 4,      /* device allocation failed */
    SDTW_E_NONFINITE = 5   /* an input sample is NaN or +-inf */
} sdtw_status;

/* Option keys for sdtw_set_option / sdtw_get_option (process-wide). */
enum {
    SDTW_OPT_NORMALIZE = 1, /* 1 (default): z-normalise reference (at set_reference) and
                               each query (§5.1 Eq. 2, "normalize both");
                               0: raw samples */
    SDTW_OPT_FMA = 2,       /* 1 (default): cell = fmaf(t,t,m); 0: fl(fl(t*t)+m) -- both
                               bit-exact with the oracle in the same mode */
    SDTW_OPT_SEGMENT_W = 3, /* reference columns per lane ("segment width"):
                               scalar 7, 15, 31; 2 chains 6, 14, 30 (default), 62; 4 chains 28, 60;
                               0 = auto */
    SDTW_OPT_LANES = 4,     /* warps per CTA in one query ring; 0 = auto */
    SDTW_OPT_CLUSTER = 5,   /* CTAs per query (thread-block cluster, DSMEM handoff); 0 = auto */
    SDTW_OPT_STREAM = 6,    /* cudaStream_t as int64 (0 = legacy default stream) */
    SDTW_OPT_PACKED = 7,    /* chains per lane: 0 = 1 (scalar FADD/FMNMX3/FFMA), 1 = 2 (one f32x2
                               FADD2/FFMA2 pair), 2 = 4 (two independent pairs); -1 = auto (2) */
    SDTW_OPT_CHUNK = 8,     /* steps between inter-warp hand-off checks, rounded to whole
                               rotation periods (WC+1 steps); 0 = auto (32) */
    SDTW_OPT_PROFILE = 9,   /* 1: time the DP kernel with CUDA events (sdtw_profile) */
    SDTW_OPT_RING = 10,     /* inter-warp hand-off ring entries (rounded up to a power of two); 0 = auto */
    SDTW_OPT_SCHED = 11,    /* 0 auto; 1 one CTA (or cluster) per query; 2 persistent CTAs pulling
                               (query, round-segment) units -- balances any Z over the SMs;
                               3 speculative segments: every round-segment of a query starts
                               at once from a +inf boundary, then a short correction pass per
                               segment boundary repairs the result exactly (also the start
                               index; fp32, no clusters, fixed-length batches; the auto
                               choice for those) */
    SDTW_OPT_SEGMENTS = 12, /* round segments per query under persistent scheduling; 0 = auto */
    SDTW_OPT_WORKERS = 13,  /* resident CTAs per SM under persistent scheduling; 0 = auto
                               (min(occupancy, n_queries / #SMs)) */
    SDTW_OPT_PAD = 15,      /* extra idle rows per round period (ring slack for long rings); 0 = auto */
    SDTW_OPT_START = 17,    /* how sdtw_traceback / sdtw_path find the start column: 0 (default)
                               auto = checkpointed when the launch qualifies, else forward;
                               1 forward propagation of the start column in every cell
                               (DESIGN.md §4 TRACE); 2 checkpointed only (SDTW_E_ARG if the
                               launch does not qualify): the cost/end DP at full speed storing
                               every round's last column, then per query a window DP from the
                               checkpoint left of its end and the paper's walk-back,
                               widened until the chain starts inside.  Both
                               give the same start (reading G6) */
    SDTW_OPT_SPEC_ROUNDS = 16, /* speculative segments: rounds of each correction pass (the
                               columns over which the boundary's paths must be overtaken by
                               the segment's own); 0 = auto (one query length of columns plus half a round, rounded up to rounds).  A segment
                               whose correction is not overtaken in time is recomputed, so
                               any value gives exact results; it only moves work */
    SDTW_OPT_PRECISION = 14,/* 32 (default): fp32 cells, bit-exact with the fp32 oracle;
                               16: packed half (the paper's __half2):
                               queries/reference rounded to binary16, every cell op rounded to
                               binary16 (HADD2, HFMA2, 3-input half2 min); costs overflow to
                               +inf above 65504;
                               8: uint8 codebook (the paper's future work P:L165;
                               DESIGN.md §16): reference and queries coded 0..255 through the
                               reference's codebook (sdtw_q8_codebook), integer cell
                               (cx - cy)^2 + min(...), optional INF pruning (SDTW_OPT_Q8_PRUNE);
                               sdtw_batch returns cost x delta^2 (delta = (hi - lo)/255) in fp32,
                               sdtw_batch_q8 the exact integer cost; N <= 12,000.
                               16 and 8: sdtw_batch / sdtw_batch_ragged / sdtw_batch_q8 only
                               (no start index), no clusters, OPT_PACKED ignored; W in {14, 30
                               (half default), 62} for 16, {14 (default), 30} for 8 */
    SDTW_OPT_Q8_PRUNE = 18, /* uint8 codebook: INF pruning of "far" cells: a cell with
                               |cx - cy| > tau is INF (2^30: no path through it); -1 (default)
                               or tau >= 255: off */
    SDTW_OPT_Q8_CLIP = 19,  /* uint8 codebook: tail mass clamped to each extreme code, in parts
                               per million of the reference (default 1000 = 0.1 %); the
                               codebook spans the order statistics of rank k and M-1-k,
                               k = floor(clip * (M-1) / 1e6) */
    SDTW_OPT_QUERY_ROWS = 21, /* where the DP kernel reads the query rows: 0 (default) auto --
                               shared memory, or for long queries a global pair-layout buffer
                               read through L1 when that keeps more CTAs resident; 1 shared
                               memory; 2 global memory (two-chain fp32 cost/end kernels and the
                               checkpointed start index; SDTW_E_ARG otherwise).  Results are
                               identical */
    SDTW_OPT_STAT_FIXUP_DEPTH = 20 /* read-only (sdtw_get_option): how many levels of speculative
                               recomputation the last call on this device needed (0: none; 1:
                               failed queries re-run once as their own speculative batch with
                               corrections x4; 2: some of those failed again; ...) */
};

/* Install the reference Y[M] on the current device (copied into a
 * library-owned, +inf-padded buffer; z-normalised globally when
 * SDTW_OPT_NORMALIZE=1).  Replaces any previous reference.  The caller may free
 * Y on return.  Errors: SDTW_E_ARG (M<1, Y NULL), SDTW_E_NONFINITE, SDTW_E_NOMEM,
 * SDTW_E_CUDA. */
sdtw_status sdtw_set_reference(const float* Y, int64_t M);

/* Batched sDTW.  Q: n_queries x N fp32, row-major, queries contiguous with no
 * gaps.  out_cost[n_queries] fp32, out_end[n_queries] int64 (0-based
 * smallest argmin column of the last row).  n_queries == 0 is a no-op.
 * Errors: SDTW_E_ARG, SDTW_E_NOREF, SDTW_E_NONFINITE, SDTW_E_NOMEM, SDTW_E_CUDA. */
sdtw_status sdtw_batch(const float* Q, int64_t n_queries, int64_t N,
                       float* out_cost, int64_t* out_end);

/* As sdtw_batch, plus out_start[n_queries] int64: the row-0 column where the
 * optimal warp path of out_end begins (P:L35 walk-back; ties diag > up > left,
 * DESIGN.md reading G6). */
sdtw_status sdtw_traceback(const float* Q, int64_t n_queries, int64_t N,
                           float* out_cost, int64_t* out_end, int64_t* out_start);

/* Ragged batch (read-until style batches of variable-length
 * reads).  Q holds the queries back to back, query q = Q[offsets[q] .. offsets[q+1]);
 * offsets: n_queries+1 int64, offsets[0] == 0, strictly increasing (every query has >= 1
 * sample); Q, offsets and the outputs may each be host or device pointers.  Per query the
 * result is exactly what sdtw_batch / sdtw_traceback return for that query alone:
 * out_cost, out_end, and out_start when out_start != NULL (start propagation on).  Each
 * query is z-normalised with its own statistics.  The DP runs all lengths in one launch
 * (per-query round period; persistent units scheduled by expected duration).
 * Errors: SDTW_E_ARG (bad offsets, OPT_PACKED 3/4), plus those of sdtw_batch. */
sdtw_status sdtw_batch_ragged(const float* Q, const int64_t* offsets, int64_t n_queries,
                              float* out_cost, int64_t* out_end, int64_t* out_start);

/* As sdtw_traceback, plus the full optimal warp path of every query (SURVEY.md
 * §8(f) NEXT-2; the walk-back of P:L35 from (N-1, out_end) with the tie rule
 * diag > up > left).  A monotone warp path visits a contiguous run of reference
 * columns in each query row, so the path is returned as path_lo / path_hi:
 * n_queries x N int32, row-major; row i of query q covers columns
 * [path_lo[q*N+i], path_hi[q*N+i]], path_lo[q*N] == out_start[q] and
 * path_hi[q*N+N-1] == out_end[q]; consecutive rows satisfy
 * path_lo[i+1] in {path_hi[i], path_hi[i]+1}.  A query whose cost is +inf (raw-mode
 * overflow) gets -1 everywhere.  Computed by re-running the DP on columns
 * [start, end] with 2-bit predecessor codes (device workspace <= 1 GiB, queries in
 * chunks).  Pointers may be host or device (current device).  Errors: as
 * sdtw_traceback; SDTW_E_NOMEM when one query's window codes exceed the workspace. */
sdtw_status sdtw_path(const float* Q, int64_t n_queries, int64_t N,
                      float* out_cost, int64_t* out_end, int64_t* out_start,
                      int32_t* path_lo, int32_t* path_hi);

/* Reference split across GPUs ("an exact reference split ...
 * boundary columns passed between GPUs").  Building blocks for
 * paper_2403_06931_b200.distributed.reference_split_batch: each rank holds one slice of
 * the (globally normalised) reference and these two calls; the Python layer exchanges the
 * columns with one all-gather.  fp32 cost/end only, fixed-length queries, no clusters.
 *
 * sdtw_round_columns: *cols = reference columns per DP round for queries of length N
 * under the current options (slice lengths and n_cols below are multiples of it).
 *
 * sdtw_batch_columns: sdtw_batch over the current reference (speculative schedule) that
 * also returns, for every query, the DP column at reference column *check_cols - 1
 * (col_check, the free DP: start anywhere in this reference, +inf left of it) and at the
 * last column M-1 (col_last; M must be a multiple of sdtw_round_columns).  Columns are
 * n_queries x N fp32 row-major DEVICE buffers (either may be NULL).
 *
 * sdtw_boundary_dp: the DP over reference columns [0, n_cols) (0 = all; else a multiple of
 * sdtw_round_columns) with left boundary column `boundary` (n_queries x N fp32, device;
 * NULL = +inf) and the free start in row 0 when free_start != 0 (else no path may start
 * here: virtual row -1 = +inf).  Returns the last-row minimum over those columns
 * (out_cost, out_end: smallest argmin; +inf / 0 when no path reaches it) and, if col_out
 * != NULL, the column n_cols - 1 (device, n_queries x N).  One DP unit per query.
 * Errors: SDTW_E_ARG (start index, ragged, half, clusters, dual-query, too few rounds for
 * the speculative schedule, bad n_cols, host column pointers), plus those of sdtw_batch. */
sdtw_status sdtw_round_columns(int64_t N, int64_t* cols);
sdtw_status sdtw_batch_columns(const float* Q, int64_t n_queries, int64_t N, float* out_cost, int64_t* out_end,
                               float* col_check, float* col_last, int64_t* check_cols);
sdtw_status sdtw_boundary_dp(const float* Q, int64_t n_queries, int64_t N, const float* boundary, int free_start,
                             int64_t n_cols, float* out_cost, int64_t* out_end, float* col_out);

/* The two decisions of the reference split, on the device, so that the
 * Python layer only moves columns and records:
 *
 * sdtw_columns_dominate: the overtaking test of the correction (DESIGN.md §13 "Why it is
 * exact": once the boundary DP is >= the free DP on a whole column it stays so on every
 * later column).  out_flag[q] = 1 iff B[q][i] >= F[q][i] for every row i < N, else 0.
 * B, F: n_queries x N fp32 row-major; out_flag: n_queries int32.  All DEVICE pointers on
 * the current device; returns after the flags are written.
 *
 * sdtw_merge_candidates: per query q, the lexicographic minimum of (cost, end) (PAPER.md
 * P:L35, the last-row minimum; reading G5: smallest end on equal cost) over the n_sets
 * candidate sets k whose valid[k][q] != 0 (valid == NULL: all valid).  cost / end /
 * valid: n_sets x n_queries, set-major; a query whose best cost is +inf gets end 0.
 * out_invalid (optional): 1 iff some set of that query was invalid (a correction that was
 * not overtaken: the query needs the exact fallback chain), else 0.  All DEVICE pointers
 * on the current device.  Errors: SDTW_E_ARG (n_sets < 1, negative sizes, NULL or host
 * pointers), SDTW_E_CUDA. */
sdtw_status sdtw_columns_dominate(const float* B, const float* F, int64_t n_queries, int64_t N, int32_t* out_flag);
sdtw_status sdtw_merge_candidates(const float* cost, const int64_t* end, const int32_t* valid, int64_t n_sets,
                                  int64_t n_queries, float* out_cost, int64_t* out_end, int32_t* out_invalid);

/* uint8-codebook sDTW (§Discussion).
 *
 * sdtw_q8_codebook: *lo, *hi = the codebook of the current reference (its order statistics of
 * rank k and M-1-k, k = floor(SDTW_OPT_Q8_CLIP * (M-1) / 1e6), of the reference as installed,
 * i.e. normalised when SDTW_OPT_NORMALIZE=1); built on first use after sdtw_set_reference.
 *
 * sdtw_quantize: out[i] = clamp(floor((in[i] - lo) * (255 / (hi - lo)) + 0.5), 0, 255), every
 * operation one fp64 rounding (hi == lo: 0).  in: n fp32, out: n bytes; host or device.
 *
 * sdtw_batch_q8: sdtw_batch with SDTW_OPT_PRECISION=8 whatever the option says, returning the
 * exact integer cost: out_cost[q] = min_j D(N-1, j) over the integer recurrence
 *     D(i,j) = INF                                    if |cx_i - cy_j| > tau (pruning on)
 *            = min((cx_i - cy_j)^2 + min(D(i-1,j), D(i,j-1), D(i-1,j-1)), INF)   otherwise,
 * INF = 2^30 (a cost of INF: every path crosses a pruned cell; out_end = 0 then);
 * out_end[q] = smallest argmin.  Queries are z-normalised first when SDTW_OPT_NORMALIZE=1,
 * then coded.  N <= 12,000 (<= 8,000 with pruning).
 * Pointers host or device.  Errors: as sdtw_batch, SDTW_E_ARG for N > 12,000. */
sdtw_status sdtw_q8_codebook(float* lo, float* hi);
sdtw_status sdtw_quantize(const float* in, int64_t n, uint8_t* out);
sdtw_status sdtw_batch_q8(const float* Q, int64_t n_queries, int64_t N, int32_t* out_cost, int64_t* out_end);

/* z-normalisation of n_series contiguous series of length len (the paper's
 * runNormalizer; Eq. 2 P:L73 with the population variance of P:L85-L86):
 * fp64 accumulation, z = fl32((x - mean)/sd); degenerate series (var <= 1e-12 *
 * E[x^2]) map to zeros.  in/out: n_series x len fp32 (may alias). */
sdtw_status sdtw_znormalize(const float* in, int64_t n_series, int64_t len, float* out);

sdtw_status sdtw_set_option(int key, int64_t value);
sdtw_status sdtw_get_option(int key, int64_t* value);

/* DP-kernel timing of the last sdtw_batch/traceback call when SDTW_OPT_PROFILE=1:
 * *dp_ms = summed CUDA-event duration of the DP kernel launch(es) on the option
 * stream; *launches = kernels the last call launched (all of them). */
sdtw_status sdtw_profile(double* dp_ms, int64_t* launches);

/* Speculative segments (SDTW_OPT_SCHED=3, or auto for small batches): *n = queries of the
 * last sdtw_batch call whose correction pass was not overtaken within OPT_SPEC_ROUNDS
 * rounds and that were therefore recomputed with sequential segments (0 otherwise). */
sdtw_status sdtw_spec_recomputed(int64_t* n);

/* Total kernels this process has launched through the library. */
int64_t sdtw_launch_count(void);

/* Thread-local text describing the last non-OK status. */
const char* sdtw_last_error(void);

/* Free the current device's context (reference, workspaces). */
void sdtw_release(void);

/* ABI version (2: exact-sum normaliser, sdtw_build_info, the reference-split merge calls). */
int sdtw_version(void);

/* Static text naming the nvcc/ptxas version the library was built with (and the float-pair
 * pack mode of the packed kernels), for bench lines and bug reports.  Owned
 * by the library; never NULL. */
const char* sdtw_build_info(void);

#ifdef __cplusplus
}
#endif
#endif /* SDTW_H */
