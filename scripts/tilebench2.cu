// tilebench2.cu -- the row-pair tile cell loop in the form a kernel would run it:
// fixed slots, no register moves.  A lane owns one strip of W columns and computes rows 2s
// (A, low half) and 2s+1 (B, high half, one column behind) per step; slot P[k] holds
// (A(2s, k), B(2s+1, k-1)).  Per micro-step k:
//   mA = min3(A(2s, k-1), B(2s-1, k-1), B(2s-1, k))  = min3(lo P[k-1], hi P[k], hi P[k+1])
//   mB = min3(A(2s, k-1), A(2s, k-2), B(2s+1, k-2))  = min3(lo P[k-1], lo P[k-2], hi P[k-1])
//   P[k] = fma2(sub2(x pair, Y pair k), same, pk(mA, mB))
// The left edges come from a SHFL per half (as the kernel's lane hand-off would).  Compared
// with the kernel's own bare loop, `scripts/mixbench.cu` packed mode (8.9-9.2 TCUPS).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tilebench2 tilebench2.cu
#include <cstdio>
#include <cuda_runtime.h>

typedef unsigned long long u64;
__device__ __forceinline__ u64 pk(float a, float b) { return ((u64)__float_as_uint(b) << 32) | __float_as_uint(a); }
__device__ __forceinline__ float lo(u64 r) { return __uint_as_float((unsigned)r); }
__device__ __forceinline__ float hi(u64 r) { return __uint_as_float((unsigned)(r >> 32)); }
__device__ __forceinline__ u64 sub2(u64 a, u64 b) { u64 r; asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ u64 fma2(u64 t, u64 m) { u64 r; asm("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(r) : "l"(t), "l"(m)); return r; }
__device__ __forceinline__ float mn3(float a, float b, float c) {
    float r;
    asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}

template <int W>
__global__ void __launch_bounds__(128) tile(float* out, int iters, float xs, long long* cyc) {
    const long long c0 = clock64();
    u64 Y[W], P[W];
#pragma unroll
    for (int k = 0; k < W; ++k) {
        Y[k] = pk(xs * k + threadIdx.x * 1e-6f, xs * (k + 1) - 1e-6f * threadIdx.x);
        P[k] = pk(1.0f + k, 2.0f + k);
    }
    float x0 = xs + threadIdx.x * 1e-5f, x1 = x0 * 0.5f;
    for (int it = 0; it < iters; ++it) {
        const u64 xx = pk(x0, x1);
        // left edges of rows 2s (A) and 2s+1 (B) from the lower lane
        const float leftA = __shfl_up_sync(0xffffffffu, hi(P[W - 1]), 1);
        float a1 = leftA, a2 = leftA;          // A(2s, k-1), A(2s, k-2)
        float bl = hi(P[0]);                   // B(2s+1, k-2) (B's left input)
#pragma unroll
        for (int k = 0; k < W; ++k) {
            const float mA = mn3(a1, hi(P[k]), hi(P[(k + 1) % W]));
            const float mB = mn3(a1, a2, bl);
            P[k] = fma2(sub2(xx, Y[k]), pk(mA, mB));
            a2 = a1;
            a1 = lo(P[k]);
            bl = hi(P[k]);
            if (k == 0) bl = __shfl_up_sync(0xffffffffu, bl, 1);     // B's left edge
        }
        x0 += 1e-7f;
        x1 -= 1e-7f;
    }
    float acc = 0.f;
#pragma unroll
    for (int k = 0; k < W; ++k) acc += lo(P[k]) + hi(P[k]);
    if (acc == 1234.5f) out[threadIdx.x] = acc;
    __syncthreads();
    if (threadIdx.x == 0) atomicMax((unsigned long long*)cyc, (unsigned long long)(clock64() - c0));
}

template <int W>
void run(int warps_per_sm) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* out;
    long long* cyc;
    cudaMalloc(&out, 4096);
    cudaMalloc(&cyc, 8);
    const int iters = 20000, block = 128, grid = sms * warps_per_sm / 4;
    tile<W><<<grid, block>>>(out, 100, 1.0f, cyc);
    cudaMemset(cyc, 0, 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    tile<W><<<grid, block>>>(out, iters, 1.0f, cyc);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    long long cy = 0;
    cudaMemcpy(&cy, cyc, 8, cudaMemcpyDeviceToHost);
    const double cells = (double)grid * block * iters * W * 2;
    printf("tile W=%2d warps/SM=%2d  %.2f TCUPS  %.1f cells/SM-cycle  clock %.0f MHz  %s\n", W, warps_per_sm,
           cells / (ms * 1e-3) / 1e12, cells / sms / (double)cy, cy / (ms * 1e-3) / 1e6,
           cudaGetErrorString(cudaGetLastError()));
    cudaFree(out);
    cudaFree(cyc);
}

int main() {
    for (int w : {8, 12, 16, 24}) {
        run<15>(w);
        run<16>(w);
        run<24>(w);
    }
    return 0;
}
