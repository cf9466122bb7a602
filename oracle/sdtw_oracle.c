/*
 * sdtw_oracle.c -- plain, slow, obviously-correct CPU oracle for batched
 * subsequence DTW (arXiv 2403.06931).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or constant with the CUDA path
 * (paper_2403_06931_b200/csrc); the product never calls it.
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -fPIC -shared -pthread
 *        (NO contraction: every fp32 operation below is separately rounded unless
 *        fmaf() is called explicitly).
 *
 * What is computed (PAPER.md line numbers as P:Lnn; readings in DESIGN.md §2):
 *
 *  Recurrence, §2 Eq. 1:
 *      D(i,j) = min{D(i-1,j), D(i,j-1), D(i-1,j-1)} + d(X_i, Y_j)
 *  with d(x,y) = (x-y)^2 (reading G2; P:L35 leaves d unspecified), evaluated
 *  in fp32 as
 *      t = fl(x - y);   FMA mode:   D = fmaf(t, t, m)          (one rounding)
 *                       NOFMA mode: D = fl(fl(t*t) + m)
 *  Subsequence initialisation ("initialized differently", reading G3):
 *  virtual row -1 is 0 (free start anywhere), virtual column -1 is +inf,
 *  D(-1,-1) = 0.
 *  Answer ("minimum valued tile in the last row"): cost = min_j D(N-1,j),
 *  end = smallest j attaining it (reading G5).
 *  Start column (P:L35 walk-back, neighbour order read as diag, up, left --
 *  reading G4/G6): S(0,j) = j; otherwise S(i,j) = S of the predecessor that
 *  attains m, priority diag > up > left on exact equality.
 *
 *  Packed half (fma_mode == 2): the same recurrence with every value
 *  rounded to binary16 after each operation (oracle_round_half / oracle_cell16 below).
 *
 *  uint8 codebook: oracle_sdtw_q8 below (exact integers).
 *
 *  The normaliser (§5.1 Eq. 2) lives in oracle/__init__.py (znorm): its
 *  sums are exact (math.fsum), which plain C fp64 accumulation is not (reading G8).
 *
 * Pins (tests/test_oracle_pins.py): SPEC worked examples, brute-force path
 * enumeration (tests/pins/brute.c), closed forms for N=1 / M=1 / constant
 * reference, embedding + time-stretch, reference-prefix, restricted-DP start
 * validity, walk-back == forward start, fp64 accuracy, normaliser fixtures.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_INF (INFINITY)

/* one cell: d(x,y) + m in fp32, P:L33 with d = (x-y)^2 */
static float oracle_cell(float x, float y, float m, int fma_mode)
{
    float t = x - y;
    if (fma_mode)
        return fmaf(t, t, m);
    float sq = t * t;
    return sq + m;
}

/* ---------------------------------------------------------------- packed half
 * SURVEY.md §8(f) NEXT-1, the paper's own precision (the fp32 queries and
 * reference are converted to float16 and processed as __half2 pairs; P:L108 __hmin2).
 * Every operation rounds to binary16 (SPEC S1: "rounds after every add/min/FMA"):
 *     x, y = half(x32), half(y32);  t = half(x - y);  D = half(t*t + m)  (one rounding,
 *     the HFMA2 of the GPU path; min is exact).
 * oracle_round_half: IEEE round-to-nearest-even to binary16 of the exact value v + err
 * (err = the exact residual of a double operation, |err| <= half a double ulp of v;
 * it only breaks exact ties), returned as a float (binary16 values are exact in fp32).
 * Overflow goes to +-inf, subnormals are kept. */
float oracle_round_half(double v, double err)
{
    if (v != v) return NAN;
    const double a = fabs(v);
    if (a == 0.0) return (float)v;
    int e;
    frexp(a, &e);                                      /* a in [2^(e-1), 2^e) */
    const double ulp = (e - 1 >= -14) ? ldexp(1.0, e - 11) : ldexp(1.0, -24);
    const double q = a / ulp;                          /* exact: power-of-two scaling */
    const double fl = floor(q), frac = q - fl;
    const double errp = (v > 0) ? err : -err;
    int up;
    if (frac > 0.5) up = 1;
    else if (frac < 0.5) up = 0;
    else up = (errp > 0) || (errp == 0 && fmod(fl, 2.0) == 1.0);
    const double r = (up ? fl + 1.0 : fl) * ulp;
    const double out = (r > 65504.0) ? INFINITY : r;
    return (float)((v < 0) ? -out : out);
}

static float oracle_cell16(float x, float y, float m)
{
    const float t = oracle_round_half((double)x - (double)y, 0.0);  /* exact in double */
    const double p = (double)t * (double)t;                          /* exact: 22 bits */
    const double s = p + (double)m;
    const double bb = s - p;                                         /* TwoSum residual */
    const double err = (p - (s - bb)) + ((double)m - bb);
    return oracle_round_half(s, err);
}

static float min3(float diag, float up, float left)
{
    float m = diag;
    if (up < m) m = up;
    if (left < m) m = left;
    return m;
}

/* ---------------------------------------------------------------- one query */
/* Column-major sweep (any order respecting the dependencies is valid; this one
 * keeps O(N) state).  prev[i] = D(i, j-1), cur[i] = D(i, j). */
static void oracle_one(const float* X, int64_t N, const float* Y, int64_t M,
                       int fma_mode, float* out_cost, int64_t* out_end,
                       int64_t* out_start, float* last_row,
                       float* prev, float* cur, int64_t* sprev, int64_t* scur)
{
    for (int64_t i = 0; i < N; ++i) { prev[i] = ORACLE_INF; sprev[i] = 0; }
    float best = ORACLE_INF;
    int64_t best_j = 0, best_s = 0;
    for (int64_t j = 0; j < M; ++j) {
        for (int64_t i = 0; i < N; ++i) {
            float up, diag, left = prev[i];
            int64_t s_up, s_diag, s_left = sprev[i];
            if (i == 0) {
                up = 0.0f; diag = 0.0f;           /* virtual row -1 */
                s_up = j; s_diag = j;
            } else {
                up = cur[i - 1]; s_up = scur[i - 1];
                diag = prev[i - 1]; s_diag = sprev[i - 1]; /* +inf at j == 0 */
            }
            float m = min3(diag, up, left);
            float v = (fma_mode == 2) ? oracle_cell16(oracle_round_half(X[i], 0.0), oracle_round_half(Y[j], 0.0), m)
                                      : oracle_cell(X[i], Y[j], m, fma_mode);
            int64_t s;
            if (i == 0) s = j;
            else if (diag == m) s = s_diag;
            else if (up == m) s = s_up;
            else s = s_left;
            cur[i] = v;
            scur[i] = s;
        }
        float last = cur[N - 1];
        if (last_row) last_row[j] = last;
        if (last < best) { best = last; best_j = j; best_s = scur[N - 1]; }
        float* tf = prev; prev = cur; cur = tf;
        int64_t* ti = sprev; sprev = scur; scur = ti;
    }
    if (M > 0 && best == ORACLE_INF) { /* only if every last-row cell overflowed */
        best_j = 0;
        best_s = 0;
    }
    *out_cost = best;
    *out_end = best_j;
    if (out_start) *out_start = best_s;
}

typedef struct {
    const float* Q; int64_t Z, N; const float* Y; int64_t M; int fma_mode;
    float* cost; int64_t* end; int64_t* start; float* last_rows;
    int64_t next; pthread_mutex_t lock;
} oracle_job;

static void* oracle_worker(void* arg)
{
    oracle_job* job = (oracle_job*)arg;
    int64_t N = job->N;
    float* prev = (float*)malloc(sizeof(float) * N);
    float* cur = (float*)malloc(sizeof(float) * N);
    int64_t* sprev = (int64_t*)malloc(sizeof(int64_t) * N);
    int64_t* scur = (int64_t*)malloc(sizeof(int64_t) * N);
    for (;;) {
        pthread_mutex_lock(&job->lock);
        int64_t q = job->next++;
        pthread_mutex_unlock(&job->lock);
        if (q >= job->Z) break;
        oracle_one(job->Q + q * N, N, job->Y, job->M, job->fma_mode,
                   &job->cost[q], &job->end[q], job->start ? &job->start[q] : NULL,
                   job->last_rows ? job->last_rows + q * job->M : NULL,
                   prev, cur, sprev, scur);
    }
    free(prev); free(cur); free(sprev); free(scur);
    return NULL;
}

/* Batched sDTW over Z queries (row-major Z x N) against Y[M].
 * start and last_rows (Z x M) may be NULL.  Returns 0 on success, 1 on bad args. */
int oracle_sdtw(const float* Q, int64_t Z, int64_t N, const float* Y, int64_t M,
                int fma_mode, float* cost, int64_t* end, int64_t* start,
                float* last_rows, int threads)
{
    if (Z < 0 || N < 1 || M < 1 || (Z > 0 && (!Q || !Y || !cost || !end))) return 1;
    if (Z == 0) return 0;
    if (threads < 1) threads = 1;
    if (threads > Z) threads = (int)Z;
    oracle_job job = {Q, Z, N, Y, M, fma_mode, cost, end, start, last_rows, 0};
    pthread_mutex_init(&job.lock, NULL);
    pthread_t* tid = (pthread_t*)malloc(sizeof(pthread_t) * threads);
    for (int t = 0; t < threads; ++t) pthread_create(&tid[t], NULL, oracle_worker, &job);
    for (int t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
    free(tid);
    pthread_mutex_destroy(&job.lock);
    return 0;
}

/* Full N x M matrices D and S (row-major) for small instances (tests only). */
int oracle_sdtw_full(const float* X, int64_t N, const float* Y, int64_t M, int fma_mode,
                     float* D, int64_t* S)
{
    if (N < 1 || M < 1) return 1;
    for (int64_t i = 0; i < N; ++i) {
        for (int64_t j = 0; j < M; ++j) {
            float up = (i == 0) ? 0.0f : D[(i - 1) * M + j];
            float left = (j == 0) ? ORACLE_INF : D[i * M + j - 1];
            float diag = (i == 0) ? 0.0f : (j == 0 ? ORACLE_INF : D[(i - 1) * M + j - 1]);
            float m = min3(diag, up, left);
            D[i * M + j] = oracle_cell(X[i], Y[j], m, fma_mode);
            int64_t s;
            if (i == 0) s = j;
            else if (diag == m) s = S[(i - 1) * M + j - 1];
            else if (up == m) s = S[(i - 1) * M + j];
            else s = S[i * M + j - 1];
            S[i * M + j] = s;
        }
    }
    return 0;
}

/* The paper's walk-back: from (N-1, end) repeatedly step to the
 * neighbour with the smallest accumulated cost among (i-1,j-1), (i-1,j),
 * (i,j-1) -- ties resolved in that order -- until row 0; returns the column. */
int64_t oracle_walkback(const float* D, int64_t N, int64_t M, int64_t end)
{
    int64_t i = N - 1, j = end;
    while (i > 0) {
        float diag = (j > 0) ? D[(i - 1) * M + j - 1] : ORACLE_INF;
        float up = D[(i - 1) * M + j];
        float left = (j > 0) ? D[i * M + j - 1] : ORACLE_INF;
        float m = min3(diag, up, left);
        if (diag == m && j > 0) { i -= 1; j -= 1; }
        else if (up == m) { i -= 1; }
        else { j -= 1; }
    }
    return j;
}

/* The full warp path: the cells the paper's walk-back
 * visits from (N-1, end) down to row 0, with the same neighbour order and tie rule
 * as oracle_walkback.  A monotone path visits a contiguous run of columns in each
 * row, so the path is reported as lo[i] <= hi[i], the first and last column it
 * visits in row i (lo[0] is the start column).  Returns 0, or 1 on bad arguments. */
int oracle_walkback_path(const float* D, int64_t N, int64_t M, int64_t end, int64_t* lo, int64_t* hi)
{
    if (N < 1 || M < 1 || end < 0 || end >= M) return 1;
    int64_t i = N - 1, j = end;
    lo[i] = hi[i] = j;
    while (i > 0) {
        float diag = (j > 0) ? D[(i - 1) * M + j - 1] : ORACLE_INF;
        float up = D[(i - 1) * M + j];
        float left = (j > 0) ? D[i * M + j - 1] : ORACLE_INF;
        float m = min3(diag, up, left);
        if (diag == m && j > 0) { i -= 1; j -= 1; hi[i] = j; }
        else if (up == m) { i -= 1; hi[i] = j; }
        else { j -= 1; }
        lo[i] = j;
    }
    return 0;
}

/* ---------------------------------------------------- uint8 codebook (NEXT-3)
 * The paper's future-work variant (§Discussion): queries and reference as
 * uint8 codes of one reference-derived codebook (the codes are made in oracle/__init__.py:
 * codebook / quantize), the cell in exact integers, and "early pruning of values that have
 * a large separation in distance": after the subtraction, a cell whose codes are more than
 * tau apart returns INF "instead of performing multiplication".  Readings:
 *     t = cx_i - cy_j;   D(i,j) = INF                               if tau >= 0 and |t| > tau
 *                               = min(t*t + min(diag, up, left), INF)  otherwise
 * INF = 2^30, the same virtual row (0) / column (INF) as the fp32 recurrence; cost = the
 * last-row minimum (a cost of INF: every path crosses a pruned cell), end = the smallest
 * column attaining it.  int64 throughout: nothing can overflow. */
#define ORACLE_Q8_INF ((int64_t)1 << 30)

static void oracle_q8_one(const uint8_t* X, int64_t N, const uint8_t* Y, int64_t M, int tau,
                          int64_t* out_cost, int64_t* out_end, int64_t* prev, int64_t* cur)
{
    for (int64_t i = 0; i < N; ++i) prev[i] = ORACLE_Q8_INF;     /* column -1 */
    int64_t best = ORACLE_Q8_INF + 1, best_j = 0;
    for (int64_t j = 0; j < M; ++j) {
        for (int64_t i = 0; i < N; ++i) {
            int64_t up = (i == 0) ? 0 : cur[i - 1];
            int64_t diag = (i == 0) ? 0 : prev[i - 1];
            int64_t left = prev[i];
            int64_t m = diag;
            if (up < m) m = up;
            if (left < m) m = left;
            int64_t t = (int64_t)X[i] - (int64_t)Y[j];
            int64_t v;
            if (tau >= 0 && (t > tau || -t > tau)) {
                v = ORACLE_Q8_INF;
            } else {
                v = t * t + m;
                if (v > ORACLE_Q8_INF) v = ORACLE_Q8_INF;
            }
            cur[i] = v;
        }
        if (cur[N - 1] < best) { best = cur[N - 1]; best_j = j; }
        int64_t* tp = prev; prev = cur; cur = tp;
    }
    *out_cost = best;
    *out_end = best_j;
}

/* Batched uint8 sDTW: Q row-major Z x N codes, Y[M] codes, tau < 0 (or >= 255): no pruning.
 * Returns 0, or 1 on bad arguments. */
int oracle_sdtw_q8(const uint8_t* Q, int64_t Z, int64_t N, const uint8_t* Y, int64_t M, int tau,
                   int64_t* cost, int64_t* end)
{
    if (Z < 0 || N < 1 || M < 1 || (Z > 0 && (!Q || !Y || !cost || !end))) return 1;
    int64_t* prev = (int64_t*)malloc(sizeof(int64_t) * N);
    int64_t* cur = (int64_t*)malloc(sizeof(int64_t) * N);
    for (int64_t q = 0; q < Z; ++q) oracle_q8_one(Q + q * N, N, Y, M, tau, &cost[q], &end[q], prev, cur);
    free(prev);
    free(cur);
    return 0;
}

int oracle_abi_version(void) { return 2; }
