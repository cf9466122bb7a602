// sdtw_prep.cuh -- z-normalisation kernels (sm_100a).
//
// PAPER.md §5.1: Eq. 2 z = (x - mean)/S with the statistics of the
// quoted code: mean = sum/n, var = sumSq/n - mean^2 (population),
// S = sqrt(var).  B200 design: one CTA per series for the batch (the paper's
// "one block is assigned to each query") and a two-pass grid reduction for
// the long reference.  Reading G8: sum and sumSq are the EXACT sums of the
// fp32 samples (x^2 is exact in fp64), each rounded once to fp64, so the result does
// not depend on the summation order and the GPU equals the oracle bit for bit.  The
// kernels accumulate in double-double (TwoSum; error-free whenever the summands' bits
// span < ~100 binades, DESIGN.md §2 G8) and round hi+lo once at the end.  Everything
// after the sums is plain fp64 with explicit _rn intrinsics (no FMA contraction of
// ex2 - mean*mean).  Degenerate series (var <= 1e-12*E[x^2] or E[x^2] == 0) map to
// zeros (reading G9).  Every kernel also raises *flag when it sees a non-finite sample
// (ABI: SDTW_E_NONFINITE).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace sdtw {

// double-double accumulator: the exact partial sum is hi + lo
struct DD { double hi, lo; };
__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
    s = __dadd_rn(a, b);
    const double bb = __dsub_rn(s, a);
    e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
}
__device__ __forceinline__ void dd_add(DD& x, double v) {
    double s, e;
    two_sum(x.hi, v, s, e);
    x.hi = s;
    x.lo = __dadd_rn(x.lo, e);
}
__device__ __forceinline__ DD dd_merge(DD a, DD b) {
    double s, e;
    two_sum(a.hi, b.hi, s, e);
    e = __dadd_rn(e, __dadd_rn(a.lo, b.lo));
    DD r;
    two_sum(s, e, r.hi, r.lo);
    return r;
}
__device__ __forceinline__ double dd_round(DD a) { return __dadd_rn(a.hi, a.lo); }

__device__ __forceinline__ DD warp_sum_dd(DD v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        DD w;
        w.hi = __shfl_xor_sync(0xffffffffu, v.hi, o);
        w.lo = __shfl_xor_sync(0xffffffffu, v.lo, o);
        v = dd_merge(v, w);
    }
    return v;
}

// Block-wide exact sums of (a, b); result valid in all threads.  scratch: 4*32 doubles.
__device__ __forceinline__ void block_sum2(DD& a, DD& b, double* scratch) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    a = warp_sum_dd(a);
    b = warp_sum_dd(b);
    __syncthreads();
    if (lane == 0) {
        scratch[warp] = a.hi; scratch[32 + warp] = a.lo;
        scratch[64 + warp] = b.hi; scratch[96 + warp] = b.lo;
    }
    __syncthreads();
    if (warp == 0) {
        DD x{0.0, 0.0}, y{0.0, 0.0};
        if (lane < nw) {
            x = DD{scratch[lane], scratch[32 + lane]};
            y = DD{scratch[64 + lane], scratch[96 + lane]};
        }
        x = warp_sum_dd(x);
        y = warp_sum_dd(y);
        if (lane == 0) { scratch[0] = x.hi; scratch[32] = x.lo; scratch[64] = y.hi; scratch[96] = y.lo; }
    }
    __syncthreads();
    a = DD{scratch[0], scratch[32]};
    b = DD{scratch[64], scratch[96]};
}

// (sum, sumsq) -> (mean, sd); false = degenerate (zeros).  Explicit _rn: no contraction.
__device__ __forceinline__ bool stats_to_affine(double sum, double sumsq, double n, double& mean,
                                                double& sd) {
    mean = __ddiv_rn(sum, n);
    const double ex2 = __ddiv_rn(sumsq, n);
    const double var = __dsub_rn(ex2, __dmul_rn(mean, mean));
    if (sumsq == 0.0 || var <= __dmul_rn(1e-12, ex2)) return false;   // degenerate -> zeros
    sd = __dsqrt_rn(var);
    return true;
}

// One CTA per series.  Normalises (normalize != 0) or only checks finiteness.
// offsets != nullptr: ragged batch, series b = in[offsets[b] .. offsets[b+1]).
__global__ void __launch_bounds__(256) znorm_rows_kernel(const float* __restrict__ in, float* out,
                                                         int64_t len, int normalize, int* flag,
                                                         const int64_t* offsets = nullptr) {
    __shared__ double scratch[128];
    int64_t base = (int64_t)blockIdx.x * len;
    if (offsets) {
        base = offsets[blockIdx.x];
        len = offsets[blockIdx.x + 1] - base;
    }
    const float* x = in + base;
    float* z = out + base;
    DD s{0.0, 0.0}, s2{0.0, 0.0};
    bool bad = false;
    for (int64_t k = threadIdx.x; k < len; k += blockDim.x) {
        const float v = x[k];
        bad |= !isfinite(v);
        const double d = (double)v;
        dd_add(s, d);
        dd_add(s2, __dmul_rn(d, d));                 // exact: 24-bit mantissa squared
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
    if (!normalize) {
        if (out != in)
            for (int64_t k = threadIdx.x; k < len; k += blockDim.x) z[k] = x[k];
        return;
    }
    block_sum2(s, s2, scratch);
    double mean, sd;
    const bool ok = stats_to_affine(dd_round(s), dd_round(s2), (double)len, mean, sd);
    for (int64_t k = threadIdx.x; k < len; k += blockDim.x)
        z[k] = ok ? (float)__ddiv_rn(__dsub_rn((double)x[k], mean), sd) : 0.0f;
}

// Reference pass 1: per-block exact partial sums (double-double: 4 doubles per block).
__global__ void __launch_bounds__(256) ref_partials_kernel(const float* __restrict__ y, int64_t M,
                                                           double* partials, int* flag) {
    __shared__ double scratch[128];
    DD s{0.0, 0.0}, s2{0.0, 0.0};
    bool bad = false;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < M;
         k += (int64_t)gridDim.x * blockDim.x) {
        const float v = y[k];
        bad |= !isfinite(v);
        const double d = (double)v;
        dd_add(s, d);
        dd_add(s2, __dmul_rn(d, d));
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
    block_sum2(s, s2, scratch);
    if (threadIdx.x == 0) {
        double* p = partials + 4 * blockIdx.x;
        p[0] = s.hi; p[1] = s.lo; p[2] = s2.hi; p[3] = s2.lo;
    }
}

// Reference pass 2: reduce partials (one CTA) -> (mean, sd, ok) in stats[0..2].
__global__ void __launch_bounds__(256) ref_stats_kernel(const double* partials, int nparts, int64_t M,
                                                        double* stats) {
    __shared__ double scratch[128];
    DD s{0.0, 0.0}, s2{0.0, 0.0};
    for (int k = threadIdx.x; k < nparts; k += blockDim.x) {
        s = dd_merge(s, DD{partials[4 * k], partials[4 * k + 1]});
        s2 = dd_merge(s2, DD{partials[4 * k + 2], partials[4 * k + 3]});
    }
    block_sum2(s, s2, scratch);
    if (threadIdx.x == 0) {
        double mean = 0.0, sd = 1.0;
        const bool ok = stats_to_affine(dd_round(s), dd_round(s2), (double)M, mean, sd);
        stats[0] = mean;
        stats[1] = sd;
        stats[2] = ok ? 1.0 : 0.0;
    }
}

// Reference pass 3: normalise (or keep raw) the padded library buffer IN PLACE; +inf pad.
// (one buffer, no __restrict__: each element is read and written by the same thread)
__global__ void __launch_bounds__(256) ref_apply_kernel(float* y, int64_t M, int64_t Malloc,
                                                        const double* stats, int normalize) {
    const double mean = stats[0], sd = stats[1];
    const bool ok = stats[2] != 0.0;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < Malloc;
         k += (int64_t)gridDim.x * blockDim.x) {
        float v;
        if (k >= M) v = INFINITY;
        else if (!normalize) continue;
        else v = ok ? (float)__ddiv_rn(__dsub_rn((double)y[k], mean), sd) : 0.0f;
        y[k] = v;
    }
}

}  // namespace sdtw
