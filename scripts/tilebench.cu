// tilebench.cu -- does pairing two ROWS of one strip (instead of two strips) cut the
// register-file cost of the packed fp32 cell? (round 2 experiment)
//
// CHAINS (the kernel's layout): a lane's f32x2 pair holds two independent chains (different
// strips); per column: FMNMX3 c0 (diag0, up0, left0), FMNMX3 c1 (diag1, up1, left1), FADD2,
// FFMA2 -- no operand shared between the two FMNMX3.
// TILE: the pair holds rows r and r+1 of the SAME strip, skewed by one column (cell (r, k) and
// (r+1, k-1) at micro-step k); both FMNMX3 read D_r[k-1] (the previous micro-step's low half),
// so with the shared operand in the same slot the second one can take it from the operand
// reuse cache.  Both loops compute W cells per row per lane-step over a rotating old row.
// Prints cells/SM/cycle and TCUPS at 148 SMs x 1965 MHz.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tilebench tilebench.cu
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

constexpr int W = 14;

template <int MODE>
__global__ void __launch_bounds__(128) bench(float* out, int iters, float xs, long long* cyc) {
    const long long c0 = clock64();
    // y of the strip (MODE 0: two strips -> pairs of different columns; MODE 1: sliding pairs)
    u64 Y[W + 1];
#pragma unroll
    for (int k = 0; k <= W; ++k) Y[k] = pk(xs * k + threadIdx.x * 1e-6f, xs * (k + 1) - 1e-6f * threadIdx.x);
    float o0[W + 1], o1[W + 1];           // old rows (row r-1 of chain 0/1, or of the tile)
#pragma unroll
    for (int k = 0; k <= W; ++k) { o0[k] = 1.0f + k; o1[k] = 2.0f + k; }
    float x0 = xs + threadIdx.x * 1e-5f, x1 = x0 * 0.5f;
    for (int it = 0; it < iters; ++it) {
        const u64 xx = pk(x0, x1);
        if (MODE == 0) {
            float l0 = o0[0], l1 = o1[0];
#pragma unroll
            for (int k = 1; k <= W; ++k) {
                const float m0 = mn3(o0[k - 1], o0[k], l0);
                const float m1 = mn3(o1[k - 1], o1[k], l1);
                const u64 v = fma2(sub2(xx, Y[k]), pk(m0, m1));
                o0[k - 1] = l0; o1[k - 1] = l1;       // rotate: old row <- new row
                l0 = lo(v); l1 = hi(v);
            }
            o0[W] = l0; o1[W] = l1;
        } else {
            // rows r (new a[]) and r+1 (new b[]) over old row o0[]; micro-step k: (r, k), (r+1, k-1)
            float a_prev = o0[0], b_prev = o1[0], a_prev2 = o1[1];
#pragma unroll
            for (int k = 1; k <= W; ++k) {
                const float mA = mn3(a_prev, o0[k - 1], o0[k]);        // shared a_prev in slot A
                const float mB = mn3(a_prev, a_prev2, b_prev);
                const u64 v = fma2(sub2(xx, Y[k]), pk(mA, mB));
                a_prev2 = a_prev;
                o0[k - 1] = b_prev;                                    // row r+1 becomes the old row
                a_prev = lo(v);
                b_prev = hi(v);
            }
            o0[W] = b_prev;
            o1[0] = a_prev;
        }
        x0 += 1e-7f; x1 -= 1e-7f;
    }
    float acc = 0.f;
#pragma unroll
    for (int k = 0; k <= W; ++k) acc += o0[k] + o1[k];
    if (acc == 1234.5f) out[threadIdx.x] = acc;
    __syncthreads();
    if (threadIdx.x == 0) atomicMax((unsigned long long*)cyc, (unsigned long long)(clock64() - c0));
}

template <int MODE>
void run(const char* name, int warps_per_sm) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* out;
    long long* cyc;
    cudaMalloc(&out, 4096);
    cudaMalloc(&cyc, 8);
    const int iters = 20000, block = 128, grid = sms * warps_per_sm / 4;
    bench<MODE><<<grid, block>>>(out, 100, 1.0f, cyc);
    cudaMemset(cyc, 0, 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    bench<MODE><<<grid, block>>>(out, iters, 1.0f, cyc);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    long long cy = 0;
    cudaMemcpy(&cy, cyc, 8, cudaMemcpyDeviceToHost);
    const double cells = (double)grid * block * iters * W * 2;
    printf("%-8s warps/SM=%2d  %.2f TCUPS  %.1f cells/SM-cycle  clock %.0f MHz  %s\n", name, warps_per_sm,
           cells / (ms * 1e-3) / 1e12, cells / sms / (double)cy, cy / (ms * 1e-3) / 1e6,
           cudaGetErrorString(cudaGetLastError()));
    cudaFree(out);
    cudaFree(cyc);
}

int main() {
    for (int w : {8, 12, 16, 24, 32}) {
        run<0>("chains", w);
        run<1>("tile", w);
    }
    return 0;
}
