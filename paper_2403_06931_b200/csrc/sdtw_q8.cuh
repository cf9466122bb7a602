// sdtw_q8.cuh -- the uint8-codebook integer variant (PAPER.md
// §Discussion: "quantize the fp16 values down to uint8 ... generating a codebook based
// on the reference string ... get the distribution of floating point values and then evenly
// divide the bulk of the distribution across uint8 values clamping any outliers to the
// extreme values", and "early pruning of values that have a large separation in distance
// ... return an infinite value (INF) instead of performing multiplication").
//
// Readings (G18-G21):
//  * codebook: lo / hi = the order statistics of rank k and M-1-k of the (normalised)
//    reference, k = floor(clip_ppm * (M-1) / 1e6) (the "bulk"); 256 equal-width levels over
//    [lo, hi] ("evenly divide"), values outside clamp to 0 / 255;
//    code(v) = clamp(floor((v - lo) * (255 / (hi - lo)) + 0.5), 0, 255), every operation one
//    IEEE fp64 rounding (no contraction); hi == lo -> every code 0.  Queries use the
//    reference's codebook.
//  * cell: t = cx - cy (integer), d = t*t; pruned (|t| > tau) -> D = INF; else
//    D = min(d + m, INF), m = min(diag, up, left), INF = 2^30 (> every finite cost: N <=
//    12,000 rows x 255^2).  Without pruning (tau >= 255) the clamp never binds on the true
//    DP (every cell has a finite vertical path from its own free start), so the kernel omits
//    it: VIMNMX3 + IADD + IMAD per cell.  With pruning the kernel computes an equivalent
//    unclamped form (kQ8Pruned below) and canonicalises the result.
//
// GPU side: the codebook is two exact order statistics found by a two-pass radix select
// (16 + 16 bits of the order-preserving key of the fp32 sample) over the reference buffer;
// the codes travel as exact small fp32 values (0..255) through the fp32 reference / query
// buffers, so the DP's staging and the schedule are the packed-half kernel's (sdtw_dp2.cuh).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "sdtw_dp2.cuh"

namespace sdtw {

constexpr int kQ8Inf = 1 << 30;
constexpr int kQ8MaxN = 12000;
// INF pruning on the GPU: a pruned cell takes kQ8Pruned = 2^29 and the others d + m without a
// clamp (5 SASS instead of a 6-SASS select + VIADDMNMX clamp, and balanced 3 ALU / 3 FMA-pipe).
// With N <= 8,000 every path that avoids pruned cells costs <= 8,000 x 255^2 < 2^29, so a
// cell's value is < 2^29 exactly when the oracle's clamped value (G20/G21) is finite, and then
// the two are equal; every true value on rows < N stays < 2^29 + 8,000 x 255^2 < 2^30 = the
// boundary INF (the speculative decomposition needs INF above every true boundary value).
// q8_canon_kernel maps a final cost >= 2^29 (every path pruned) to the oracle's (INF, end 0).
constexpr int kQ8Pruned = 1 << 29;
constexpr int kQ8PruneMaxN = 8000;

struct I2 { int a, b; };   // one column of both chains

template <bool PRUNE>
struct Q8Arith {
    using V = I2;
    using S = int;
    using XW = int2;
    static constexpr int kSBytes = 4, kXWBytes = 8;
    static constexpr bool kMaskPad = true;     // padded columns hold code 0: excluded from the fold
    __device__ static __forceinline__ S inf() { return kQ8Inf; }
    __device__ static __forceinline__ S zero() { return 0; }
    __device__ static __forceinline__ V splat(S v) { return I2{v, v}; }
    __device__ static __forceinline__ V with(V p, int c, S v) { return c ? I2{p.a, v} : I2{v, p.b}; }
    __device__ static __forceinline__ S get(V p, int c) { return c ? p.b : p.a; }
    __device__ static __forceinline__ XW xword(float a, float b) { return make_int2((int)a, (int)b); }
    __device__ static __forceinline__ V xval(XW w) { return I2{w.x, w.y}; }
    // staged codes; columns past the padded buffer arrive as +inf: code 0 (masked anyway)
    __device__ static __forceinline__ S yval(float y) { return y < 256.0f ? (int)y : 0; }
    __device__ static __forceinline__ V left_in(V right, S e, bool use_in) {
        const int s = __shfl_up_sync(0xffffffffu, right.b, 1);
        return I2{use_in ? e : s, right.a};
    }
    __device__ static __forceinline__ int one(int dg, int up, int left, int x, int y, int tau2) {
        const int m = __vimin3_s32(dg, up, left);
        const int t = x - y;
        if constexpr (!PRUNE) {
            return t * t + m;
        } else {
            // pruned: the fixed value 2^29 (not INF + m: no growth along pruned chains), else
            // d + m unclamped -- see kQ8Pruned; the host canonicalises costs >= 2^29 to INF
            const int d = t * t;
            return d > tau2 ? kQ8Pruned : d + m;
        }
    }
    __device__ static __forceinline__ V cell(V dg, V up, V left, V xx, V y, int tau2) {
        return I2{one(dg.a, up.a, left.a, xx.a, y.a, tau2), one(dg.b, up.b, left.b, xx.b, y.b, tau2)};
    }
    // order-preserving fp32 image: 0 <= v < 2^31 - 2^23 -> a finite non-negative float
    __device__ static __forceinline__ float key(S v) { return __int_as_float(v); }
};

// ------------------------------------------------------------------ codebook
// Order-preserving 32-bit key of an fp32 value (finite inputs).
__device__ __forceinline__ unsigned q8_key(float v) {
    const unsigned u = __float_as_uint(v);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float q8_unkey(unsigned k) {
    return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

// pass 0: histogram of the high 16 key bits; pass 1: of the low 16 bits among the samples
// whose high half equals sel[j].hi, one histogram per wanted rank j (2 ranks)
struct Q8Sel { unsigned hi; unsigned rank; unsigned key; unsigned pad; };

static __global__ void __launch_bounds__(256) q8_hist_kernel(const float* __restrict__ y, int64_t M, unsigned* hist,
                                                      const Q8Sel* sel, int pass) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < M; i += stride) {
        const unsigned k = q8_key(y[i]);
        if (pass == 0) {
            atomicAdd(hist + (k >> 16), 1u);
        } else {
#pragma unroll
            for (int j = 0; j < 2; ++j)
                if ((k >> 16) == sel[j].hi) atomicAdd(hist + j * 65536 + (k & 0xffffu), 1u);
        }
    }
}

// One block of 1024 threads: find, for each wanted rank, the bin that holds it (prefix
// sums over 65,536 bins) and the rank left inside that bin.  pass 0 sets sel[j].hi and
// sel[j].rank (the remaining rank); pass 1 sets sel[j].key (the full key).
static __global__ void __launch_bounds__(1024) q8_select_kernel(const unsigned* hist, Q8Sel* sel, int pass,
                                                        unsigned rank_lo, unsigned rank_hi) {
    __shared__ unsigned wsum[32];
    for (int j = 0; j < 2; ++j) {
        const unsigned* h = hist + (pass == 0 ? 0 : j * 65536);
        const unsigned want = pass == 0 ? (j == 0 ? rank_lo : rank_hi) : sel[j].rank;
        const int t = threadIdx.x;
        unsigned s = 0;
        for (int b = 0; b < 64; ++b) s += h[t * 64 + b];
        // exclusive prefix over threads
        const int lane = t & 31, w = t >> 5;
        unsigned inc = s;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned n = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += n;
        }
        if (lane == 31) wsum[w] = inc;
        __syncthreads();
        if (w == 0) {
            unsigned v = wsum[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned n = __shfl_up_sync(0xffffffffu, v, o);
                if (lane >= o) v += n;
            }
            wsum[lane] = v;
        }
        __syncthreads();
        const unsigned before = inc - s + (w > 0 ? wsum[w - 1] : 0u);
        __syncthreads();
        if (want >= before && want < before + s) {          // exactly one thread
            unsigned acc = before;
            for (int b = 0; b < 64; ++b) {
                const unsigned c = h[t * 64 + b];
                if (want < acc + c) {
                    const unsigned bin = (unsigned)(t * 64 + b);
                    if (pass == 0) { sel[j].hi = bin; sel[j].rank = want - acc; }
                    else sel[j].key = (sel[j].hi << 16) | bin;
                    break;
                }
                acc += c;
            }
        }
        __syncthreads();
    }
}

// codebook[0] = lo, codebook[1] = hi (fp32 values of the two order statistics)
static __global__ void q8_codebook_kernel(const Q8Sel* sel, float* codebook) {
    if (threadIdx.x == 0) {
        codebook[0] = q8_unkey(sel[0].key);
        codebook[1] = q8_unkey(sel[1].key);
    }
}

__device__ __forceinline__ float q8_code(float v, double lo, double hi) {
    if (!(hi > lo)) return 0.0f;
    const double s = __ddiv_rn(255.0, __dsub_rn(hi, lo));
    const double u = __dadd_rn(__dmul_rn(__dsub_rn((double)v, lo), s), 0.5);
    double c = floor(u);
    c = c < 0.0 ? 0.0 : (c > 255.0 ? 255.0 : c);
    return (float)c;
}

// codes of in[0..n) as exact fp32 values 0..255 (out[n..npad) = 0: padded columns)
static __global__ void __launch_bounds__(256) q8_quantize_kernel(const float* __restrict__ in, int64_t n, int64_t npad,
                                                          const float* __restrict__ codebook, float* out) {
    const double lo = codebook[0], hi = codebook[1];
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < npad; i += stride)
        out[i] = i < n ? q8_code(in[i], lo, hi) : 0.0f;
}

// sdtw_quantize: raise *flag on a non-finite sample (no codes are returned then)
static __global__ void __launch_bounds__(256) finite_check_kernel(const float* __restrict__ in, int64_t n, int* flag) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    bool bad = false;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) bad |= !isfinite(in[i]);
    if (bad) atomicOr(flag, 1);
}

// the same codes as bytes (sdtw_quantize)
static __global__ void __launch_bounds__(256) q8_codes_u8_kernel(const float* __restrict__ in, int64_t n,
                                                          const float* __restrict__ codebook, unsigned char* out) {
    const double lo = codebook[0], hi = codebook[1];
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        out[i] = (unsigned char)q8_code(in[i], lo, hi);
}

// INF pruning: a cost >= kQ8Pruned means every path crosses a pruned cell -> (INF, end 0)
static __global__ void q8_canon_kernel(float* cost, int64_t* end, int64_t n, const int* err) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || *err) return;
    if (__float_as_int(cost[i]) >= kQ8Pruned) {
        cost[i] = __int_as_float(kQ8Inf);
        end[i] = 0;
    }
}

// sdtw_batch at OPT_PRECISION=8: the integer cost (carried as fp32 bits) scaled back to
// the normalised units, cost * delta^2 with delta = (hi - lo) / 255, rounded once to fp32;
// INF (no path survived the pruning) -> +inf
static __global__ void q8_scale_kernel(float* cost, int64_t n, const float* __restrict__ codebook, const int* err) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || *err) return;
    const int v = __float_as_int(cost[i]);
    const double delta = __ddiv_rn(__dsub_rn((double)codebook[1], (double)codebook[0]), 255.0);
    cost[i] = v >= kQ8Inf ? INFINITY : (float)__dmul_rn((double)v, __dmul_rn(delta, delta));
}

}  // namespace sdtw
