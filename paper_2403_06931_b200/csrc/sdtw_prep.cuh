// sdtw_prep.cuh -- z-normalisation kernels (sm_100a).
//
// PAPER.md §5.1: Eq. 2 z = (x - mean)/S with the statistics of the
// quoted code: mean = sum/n, var = sumSq/n - mean^2 (population),
// S = sqrt(var).  B200 design: one CTA per series for the batch (the paper's
// "one block is assigned to each query") but fp64 accumulation with warp
// shuffles instead of an fp32 shared-memory tree (reading G8), and a
// two-pass grid reduction for the long reference.  Degenerate series
// (var <= 1e-12*E[x^2] or E[x^2] == 0) map to zeros (reading G9).  Every kernel
// also raises *flag when it sees a non-finite sample (ABI: SDTW_E_NONFINITE).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace sdtw {

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Block-wide sum of (a, b); result valid in all threads.  scratch: 2*32 doubles.
__device__ __forceinline__ void block_sum2(double& a, double& b, double* scratch) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    a = warp_sum_d(a);
    b = warp_sum_d(b);
    __syncthreads();
    if (lane == 0) { scratch[warp] = a; scratch[32 + warp] = b; }
    __syncthreads();
    if (warp == 0) {
        double x = (lane < nw) ? scratch[lane] : 0.0;
        double y = (lane < nw) ? scratch[32 + lane] : 0.0;
        x = warp_sum_d(x);
        y = warp_sum_d(y);
        if (lane == 0) { scratch[0] = x; scratch[32] = y; }
    }
    __syncthreads();
    a = scratch[0];
    b = scratch[32];
}

__device__ __forceinline__ bool stats_to_affine(double sum, double sumsq, double n, double& mean,
                                                double& sd) {
    mean = sum / n;
    const double ex2 = sumsq / n;
    const double var = ex2 - mean * mean;
    if (sumsq == 0.0 || var <= 1e-12 * ex2) return false;   // degenerate -> zeros
    sd = sqrt(var);
    return true;
}

// One CTA per series.  Normalises (normalize != 0) or only checks finiteness.
// offsets != nullptr: ragged batch, series b = in[offsets[b] .. offsets[b+1]).
__global__ void __launch_bounds__(256) znorm_rows_kernel(const float* __restrict__ in, float* out,
                                                         int64_t len, int normalize, int* flag,
                                                         const int64_t* offsets = nullptr) {
    __shared__ double scratch[64];
    int64_t base = (int64_t)blockIdx.x * len;
    if (offsets) {
        base = offsets[blockIdx.x];
        len = offsets[blockIdx.x + 1] - base;
    }
    const float* x = in + base;
    float* z = out + base;
    double s = 0.0, s2 = 0.0;
    bool bad = false;
    for (int64_t k = threadIdx.x; k < len; k += blockDim.x) {
        const float v = x[k];
        bad |= !isfinite(v);
        const double d = (double)v;
        s += d;
        s2 += d * d;
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
    if (!normalize) {
        if (out != in)
            for (int64_t k = threadIdx.x; k < len; k += blockDim.x) z[k] = x[k];
        return;
    }
    block_sum2(s, s2, scratch);
    double mean, sd;
    const bool ok = stats_to_affine(s, s2, (double)len, mean, sd);
    for (int64_t k = threadIdx.x; k < len; k += blockDim.x)
        z[k] = ok ? (float)(((double)x[k] - mean) / sd) : 0.0f;
}

// Reference pass 1: per-block fp64 partial sums (deterministic order per block).
__global__ void __launch_bounds__(256) ref_partials_kernel(const float* __restrict__ y, int64_t M,
                                                           double* partials, int* flag) {
    __shared__ double scratch[64];
    double s = 0.0, s2 = 0.0;
    bool bad = false;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < M;
         k += (int64_t)gridDim.x * blockDim.x) {
        const float v = y[k];
        bad |= !isfinite(v);
        const double d = (double)v;
        s += d;
        s2 += d * d;
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
    block_sum2(s, s2, scratch);
    if (threadIdx.x == 0) { partials[2 * blockIdx.x] = s; partials[2 * blockIdx.x + 1] = s2; }
}

// Reference pass 2: reduce partials (one CTA) -> (mean, sd, ok) in stats[0..2].
__global__ void __launch_bounds__(256) ref_stats_kernel(const double* partials, int nparts, int64_t M,
                                                        double* stats) {
    __shared__ double scratch[64];
    double s = 0.0, s2 = 0.0;
    for (int k = threadIdx.x; k < nparts; k += blockDim.x) { s += partials[2 * k]; s2 += partials[2 * k + 1]; }
    block_sum2(s, s2, scratch);
    if (threadIdx.x == 0) {
        double mean = 0.0, sd = 1.0;
        const bool ok = stats_to_affine(s, s2, (double)M, mean, sd);
        stats[0] = mean;
        stats[1] = sd;
        stats[2] = ok ? 1.0 : 0.0;
    }
}

// Reference pass 3: apply (or copy raw) into the padded library buffer; +inf pad.
__global__ void __launch_bounds__(256) ref_apply_kernel(const float* __restrict__ y, int64_t M,
                                                        int64_t Malloc, const double* stats,
                                                        int normalize, float* out) {
    const double mean = stats[0], sd = stats[1];
    const bool ok = stats[2] != 0.0;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < Malloc;
         k += (int64_t)gridDim.x * blockDim.x) {
        float v;
        if (k >= M) v = INFINITY;
        else if (!normalize) v = y[k];
        else v = ok ? (float)(((double)y[k] - mean) / sd) : 0.0f;
        out[k] = v;
    }
}

}  // namespace sdtw
