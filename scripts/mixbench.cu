// mixbench.cu -- throughput of the sDTW cell's instruction mixes on one B200 SM type
// (round 2: which mix of FADD/FADD2, FFMA/FFMA2 and FMNMX3 issues fastest when the
// dependency chains are NOT the limit).  Every variant computes the same recurrence-shaped
// work per cell: m = min3(d, u, l); t = x - y; v = t*t + m, for ILP independent cell chains
// per thread; 2 cells per "pair".  Prints cells/cycle/SM and the equivalent TCUPS at 148 SMs
// x 1965 MHz.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mixbench mixbench.cu
#include <cstdio>
#include <cuda_runtime.h>

typedef unsigned long long u64;
__device__ __forceinline__ u64 pk(float a, float b) {
    return ((u64)__float_as_uint(b) << 32) | __float_as_uint(a);
}
__device__ __forceinline__ float lo(u64 r) { return __uint_as_float((unsigned)r); }
__device__ __forceinline__ float hi(u64 r) { return __uint_as_float((unsigned)(r >> 32)); }
__device__ __forceinline__ u64 sub2(u64 a, u64 b) { u64 r; asm volatile("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ u64 fma2(u64 a, u64 c) { u64 r; asm volatile("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(r) : "l"(a), "l"(c)); return r; }
__device__ __forceinline__ float min3(float a, float b, float c) { return fminf(fminf(a, b), c); }

// MODE 0: packed  (FADD2 + FFMA2 + 2 FMNMX3 per pair)
// MODE 1: scalar  (2 FADD + 2 FFMA + 2 FMNMX3)
// MODE 2: FADD2 + 2 FFMA + 2 FMNMX3
// MODE 3: 2 FADD + FFMA2 + 2 FMNMX3
// MODE 4: FMNMX3 alone (2 per pair)
// MODE 5: FFMA2 alone
// MODE 6: FADD2 alone
template <int MODE, int ILP>
__global__ void bench(float* out, int iters, float xs, float ys, long long* cyc) {
    const long long c0 = clock64();
    u64 st[ILP], up[ILP];
    float x0 = xs + threadIdx.x * 1e-7f, x1 = x0 + 1e-7f;
    const u64 x = pk(x0, x1);
#pragma unroll
    for (int k = 0; k < ILP; ++k) { st[k] = pk(ys + k, ys - k); up[k] = pk(ys * k, ys + 2 * k); }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < ILP; ++k) {
            // chain k: st[k] = the last cell pair (up/left), up[k] = the one before (diag)
            const u64 d = up[k], u = st[k];
            if (MODE == 4) {
                const float m0 = min3(lo(d), lo(u), hi(d)), m1 = min3(hi(d), hi(u), lo(d));
                up[k] = u; st[k] = pk(m1, m0);
                continue;
            }
            if (MODE == 5) { st[k] = fma2(st[k], up[k]); continue; }
            if (MODE == 6) { st[k] = sub2(st[k], x); continue; }
            const float m0 = min3(lo(d), lo(u), hi(d));
            const float m1 = min3(hi(d), hi(u), lo(d));
            u64 v;
            if (MODE == 0) {
                const u64 t = sub2(x, u);
                v = fma2(t, pk(m0, m1));
            } else if (MODE == 1) {
                const float t0 = x0 - lo(u), t1 = x1 - hi(u);
                v = pk(__fmaf_rn(t0, t0, m0), __fmaf_rn(t1, t1, m1));
            } else if (MODE == 2) {
                const u64 t = sub2(x, u);
                v = pk(__fmaf_rn(lo(t), lo(t), m0), __fmaf_rn(hi(t), hi(t), m1));
            } else {
                const float t0 = x0 - lo(u), t1 = x1 - hi(u);
                v = fma2(pk(t0, t1), pk(m0, m1));
            }
            up[k] = u;
            st[k] = v;
        }
    }
    float acc = 0.f;
#pragma unroll
    for (int k = 0; k < ILP; ++k) acc += lo(st[k]) + hi(up[k]);
    if (acc == 1234.5f) out[threadIdx.x] = acc;
    __syncthreads();
    if (threadIdx.x == 0) atomicMax((unsigned long long*)cyc, (unsigned long long)(clock64() - c0));
}

template <int MODE, int ILP>
void run(const char* name, int warps_per_sm) {
    int dev = 0, sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    float* out;
    cudaMalloc(&out, 4096);
    long long* cyc;
    cudaMalloc(&cyc, 8);
    const int iters = 32768;
    const int block = 128;                      // 4 warps per CTA
    const int grid = sms * warps_per_sm / 4;
    bench<MODE, ILP><<<grid, block>>>(out, 2048, 1.0f, 2.0f, cyc);
    cudaMemset(cyc, 0, 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    bench<MODE, ILP><<<grid, block>>>(out, iters, 1.0f, 2.0f, cyc);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    long long cy = 0;
    cudaMemcpy(&cy, cyc, 8, cudaMemcpyDeviceToHost);
    const double cells = (double)grid * block * iters * ILP * 2;   // 2 cells per pair
    const double tcups = cells / (ms * 1e-3) / 1e12;
    // all CTAs are co-resident (one wave): SM cycles of the slowest CTA = the kernel's cycles
    printf("%-34s ILP=%d warps/SM=%2d  %.2f TCUPS  %.1f cells/SM-cycle  clock %.0f MHz  err=%s\n", name, ILP,
           warps_per_sm, tcups, cells / sms / (double)cy, cy / (ms * 1e-3) / 1e6,
           cudaGetErrorString(cudaGetLastError()));
    cudaFree(out);
    cudaFree(cyc);
}

int main() {
    for (int w : {8, 16, 24, 32}) {
        run<0, 4>("packed FADD2+FFMA2+2xFMNMX3", w);
        run<1, 4>("scalar 2xFADD+2xFFMA+2xFMNMX3", w);
        run<2, 4>("FADD2+2xFFMA+2xFMNMX3", w);
        run<3, 4>("2xFADD+FFMA2+2xFMNMX3", w);
    }
    for (int w : {16, 32}) {
        run<0, 1>("packed ILP1", w);
        run<0, 2>("packed ILP2", w);
        run<2, 1>("FADD2+2xFFMA ILP1", w);
        run<2, 2>("FADD2+2xFFMA ILP2", w);
        run<1, 2>("scalar ILP2", w);
        run<4, 4>("FMNMX3 only (2/pair)", w);
        run<5, 4>("FFMA2 only (1/pair)", w);
        run<6, 4>("FADD2 only (1/pair)", w);
    }
    return 0;
}
