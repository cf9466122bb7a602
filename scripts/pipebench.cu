// pipebench.cu -- throughput / latency of the DP's SASS ops on this GPU (B200, sm_100a).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipebench pipebench.cu
// Each kernel runs ILP independent chains per thread; per-SM ops/cycle are derived from
// clock64 and the op count.  ILP=1 gives the dependent-chain latency.
#include <cstdio>
#include <cuda_runtime.h>

#define REPS 4096

__device__ __forceinline__ unsigned long long pk(float a, float b) {
    unsigned long long r;
    asm volatile("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}

template <int OP, int ILP>
__global__ void bench(float* out, long long* cyc, float s) {
    float a[ILP], b = s * 0.5f + 1.0f, c = s * 0.25f + 2.0f;
    unsigned long long p[ILP], q = pk(b, c), r2 = pk(c, b);
#pragma unroll
    for (int k = 0; k < ILP; ++k) { a[k] = s + k; p[k] = pk(s + k, s - k); }
    __syncthreads();
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < REPS; ++i) {
#pragma unroll
        for (int k = 0; k < ILP; ++k) {
            if (OP == 0) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[k]) : "f"(b), "f"(c));
            if (OP == 1) asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(a[k]) : "f"(b));
            if (OP == 2) asm volatile("min.f32 %0, %0, %1, %2;" : "+f"(a[k]) : "f"(b), "f"(c));
            if (OP == 3) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p[k]) : "l"(q), "l"(r2));
            if (OP == 4) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(p[k]) : "l"(q));
            if (OP == 5) asm volatile("min.f32 %0, %0, %1;" : "+f"(a[k]) : "f"(b));
            if (OP == 6) {  // the DP cell pair: FADD2, 2x FMNMX3, FFMA2 (chain through p[k])
                unsigned long long t;
                float lo, hi;
                asm volatile("sub.rn.f32x2 %0, %1, %2;" : "=l"(t) : "l"(q), "l"(r2));
                asm volatile("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(p[k]));
                asm volatile("min.f32 %0, %0, %1, %2;" : "+f"(lo) : "f"(b), "f"(c));
                asm volatile("min.f32 %0, %0, %1, %2;" : "+f"(hi) : "f"(c), "f"(b));
                asm volatile("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(p[k]) : "l"(t), "l"(pk(lo, hi)));
            }
            if (OP == 7) {  // the scalar DP cell: FADD, FMNMX3, FFMA (chain through a[k])
                float t;
                asm volatile("sub.rn.f32 %0, %1, %2;" : "=f"(t) : "f"(b), "f"(c));
                asm volatile("min.f32 %0, %0, %1, %2;" : "+f"(a[k]) : "f"(b), "f"(c));
                asm volatile("fma.rn.f32 %0, %1, %1, %0;" : "+f"(a[k]) : "f"(t));
            }
        }
    }
    long long t1 = clock64();
    float acc = 0;
#pragma unroll
    for (int k = 0; k < ILP; ++k) {
        float lo, hi;
        asm volatile("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(p[k]));
        acc += a[k] + lo + hi;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP, int ILP>
void run(const char* name, int ops_per_iter, int warps_per_sm) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int threads = 32 * warps_per_sm;
    float* out;
    long long* cyc;
    cudaMalloc(&out, sizeof(float) * sms * threads);
    cudaMalloc(&cyc, sizeof(long long) * sms);
    bench<OP, ILP><<<sms, threads>>>(out, cyc, 1.0f);
    cudaDeviceSynchronize();
    bench<OP, ILP><<<sms, threads>>>(out, cyc, 1.0f);
    cudaDeviceSynchronize();
    long long h = 0;
    cudaMemcpy(&h, cyc, sizeof(long long), cudaMemcpyDeviceToHost);
    const double warp_instr = (double)REPS * ILP * ops_per_iter * warps_per_sm;  // per SM
    printf("%-26s ILP=%d warps/SM=%2d  cycles/iter/warp=%7.2f  warp-instr/cycle/SM=%5.2f\n", name, ILP,
           warps_per_sm, (double)h / REPS / ILP, warp_instr / (double)h);
    cudaFree(out);
    cudaFree(cyc);
}

int main() {
    // latency (1 warp, 1 chain) and throughput (many warps, 8 chains)
    run<0, 1>("FFMA", 1, 1);        run<0, 8>("FFMA", 1, 32);
    run<1, 1>("FADD", 1, 1);        run<1, 8>("FADD", 1, 32);
    run<2, 1>("FMNMX3 (min3)", 1, 1); run<2, 8>("FMNMX3 (min3)", 1, 32);
    run<5, 1>("FMNMX (min2)", 1, 1); run<5, 8>("FMNMX (min2)", 1, 32);
    run<3, 1>("FFMA2", 1, 1);       run<3, 8>("FFMA2", 1, 32);
    run<4, 1>("FADD2", 1, 1);       run<4, 8>("FADD2", 1, 32);
    run<6, 1>("DP pair (4 instr)", 4, 1);
    run<6, 1>("DP pair (4 instr)", 4, 4);
    run<6, 1>("DP pair (4 instr)", 4, 8);
    run<6, 1>("DP pair (4 instr)", 4, 16);
    run<6, 2>("DP pair (4 instr)", 4, 8);
    run<6, 2>("DP pair (4 instr)", 4, 16);
    run<6, 4>("DP pair (4 instr)", 4, 16);
    run<6, 8>("DP pair (4 instr)", 4, 32);
    run<7, 1>("DP scalar (3 instr)", 3, 1);
    run<7, 1>("DP scalar (3 instr)", 3, 16);
    run<7, 2>("DP scalar (3 instr)", 3, 16);
    run<7, 8>("DP scalar (3 instr)", 3, 32);
    return 0;
}
