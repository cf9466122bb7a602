/*
 * brute.c -- independent pins for the oracle (tests only; shares no code with
 * oracle/ or the CUDA path).
 *
 * brute_sdtw: minimum, over EVERY monotone warp path that starts anywhere in
 *   row 0 and ends anywhere in row N-1 (steps right, down, diagonal -- the
 *   three neighbours of PAPER.md Eq. 1), of the path's left-fold cost
 *       c_0 = cell(x_0, y_s, 0),  c_k = cell(x_i, y_j, c_{k-1})
 *   where cell is the same single fp32 cell evaluation as the definition
 *   (t = x-y; FMA: fmaf(t,t,c); NOFMA: fl(fl(t*t)+c)).  Because fl(a+.) and
 *   fmaf(t,t,.) are monotone, min-then-add equals the min over paths, so the
 *   DP must agree BIT FOR BIT.  Reports the smallest end column attaining it.
 *
 * restricted_dp: the DP with row 0 free ONLY at column s (every other row-0
 *   start is +inf).  A correct start index s for (cost, end) must reproduce
 *   exactly `cost` at column `end` (SURVEY.md §8(c) start-validity pin).
 *
 * Build: gcc -O2 -ffp-contract=off -fno-fast-math -shared -fPIC
 */
#include <math.h>
#include <stdint.h>

static float bcell(float x, float y, float c, int fma_mode)
{
    float t = x - y;
    if (fma_mode) return fmaf(t, t, c);
    float sq = t * t;
    return sq + c;
}

static void dfs(const float* X, int64_t N, const float* Y, int64_t M, int fma_mode,
                int64_t i, int64_t j, float c, float* best_per_col)
{
    if (i == N - 1 && c < best_per_col[j]) best_per_col[j] = c;
    if (j + 1 < M) dfs(X, N, Y, M, fma_mode, i, j + 1, bcell(X[i], Y[j + 1], c, fma_mode), best_per_col);
    if (i + 1 < N) dfs(X, N, Y, M, fma_mode, i + 1, j, bcell(X[i + 1], Y[j], c, fma_mode), best_per_col);
    if (i + 1 < N && j + 1 < M)
        dfs(X, N, Y, M, fma_mode, i + 1, j + 1, bcell(X[i + 1], Y[j + 1], c, fma_mode), best_per_col);
}

/* best_per_col[M] receives the brute-force last row; returns via out_cost/out_end */
void brute_sdtw(const float* X, int64_t N, const float* Y, int64_t M, int fma_mode,
                float* best_per_col, float* out_cost, int64_t* out_end)
{
    for (int64_t j = 0; j < M; ++j) best_per_col[j] = INFINITY;
    for (int64_t s = 0; s < M; ++s)
        dfs(X, N, Y, M, fma_mode, 0, s, bcell(X[0], Y[s], 0.0f, fma_mode), best_per_col);
    float best = INFINITY;
    int64_t e = 0;
    for (int64_t j = 0; j < M; ++j)
        if (best_per_col[j] < best) { best = best_per_col[j]; e = j; }
    *out_cost = best;
    *out_end = e;
}

/* Row-major rolling DP restricted to start column s; returns D(N-1, end). */
float restricted_dp(const float* X, int64_t N, const float* Y, int64_t M, int fma_mode,
                    int64_t s, int64_t end, float* row_a, float* row_b)
{
    float* prev = row_a;
    float* cur = row_b;
    for (int64_t j = 0; j < M; ++j) prev[j] = INFINITY;
    for (int64_t i = 0; i < N; ++i) {
        for (int64_t j = 0; j < M; ++j) {
            float m;
            if (i == 0) {
                /* only column s may begin a path (from the virtual zero row) */
                float left = (j > 0) ? cur[j - 1] : INFINITY;
                m = (j == s) ? 0.0f : left;
                if (j < s) { cur[j] = INFINITY; continue; }
            } else {
                float up = prev[j];
                float diag = (j > 0) ? prev[j - 1] : INFINITY;
                float left = (j > 0) ? cur[j - 1] : INFINITY;
                m = diag;
                if (up < m) m = up;
                if (left < m) m = left;
            }
            cur[j] = (m == INFINITY) ? INFINITY : bcell(X[i], Y[j], m, fma_mode);
        }
        float* t = prev; prev = cur; cur = t;
    }
    return prev[end];
}
