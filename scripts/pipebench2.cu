// pipebench2.cu -- whole-GPU throughput of the DP cell instruction mixes on B200,
// timed with CUDA events (cells/s), for ILP (independent chains per thread) x
// warps per SM.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipebench2 pipebench2.cu
#include <cstdio>
#include <cuda_runtime.h>

#define REPS 2048
#define WCELLS 16   // cells per chain per "step" (like a strip)

__device__ __forceinline__ unsigned long long pk(float a, float b) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ float lo(unsigned long long r) { float a, b; asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(r)); return a; }
__device__ __forceinline__ float hi(unsigned long long r) { float a, b; asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(r)); return b; }

// MODE 0: scalar cells (FADD, FMNMX3, FFMA); MODE 1: packed pairs (FADD2, 2 FMNMX3, FFMA2)
template <int MODE, int ILP>
__global__ void dp(float* out, float x0) {
    float up[ILP][WCELLS], y[WCELLS];
    float left[ILP];
#pragma unroll
    for (int w = 0; w < WCELLS; ++w) y[w] = x0 * w;
#pragma unroll
    for (int k = 0; k < ILP; ++k) {
        left[k] = k;
#pragma unroll
        for (int w = 0; w < WCELLS; ++w) up[k][w] = w + k;
    }
    const float x = x0 + threadIdx.x;
#pragma unroll 1
    for (int it = 0; it < REPS; ++it) {
#pragma unroll
        for (int k = 0; k < ILP; ++k) {
            if (MODE == 0) {
                float l = left[k], d = left[k];
#pragma unroll
                for (int w = 0; w < WCELLS; ++w) {
                    const float u = up[k][w];
                    const float m = fminf(fminf(d, u), l);
                    const float t = __fsub_rn(x, y[w]);
                    const float v = __fmaf_rn(t, t, m);
                    d = u; up[k][w] = v; l = v;
                }
                left[k] = l * 0.5f;
            } else {
                // pairs: chain (k, k') packed; WCELLS cells per half
                float l0 = left[k], l1 = left[k] + 1.f, d0 = l0, d1 = l1;
#pragma unroll
                for (int w = 0; w < WCELLS; w += 2) {
                    const float u0 = up[k][w], u1 = up[k][w + 1];
                    const float m0 = fminf(fminf(d0, u0), l0);
                    const float m1 = fminf(fminf(d1, u1), l1);
                    unsigned long long tt, vv;
                    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(tt) : "l"(pk(x, x + 1.f)), "l"(pk(y[w], y[w + 1])));
                    asm("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(vv) : "l"(tt), "l"(pk(m0, m1)));
                    d0 = u0; d1 = u1;
                    up[k][w] = lo(vv); up[k][w + 1] = hi(vv);
                    l0 = lo(vv); l1 = hi(vv);
                }
                left[k] = fminf(l0, l1) * 0.5f;
            }
        }
    }
    float acc = 0;
#pragma unroll
    for (int k = 0; k < ILP; ++k)
#pragma unroll
        for (int w = 0; w < WCELLS; ++w) acc += up[k][w];
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int MODE, int ILP>
void run(int warps_per_sm) {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* out;
    cudaMalloc(&out, sizeof(float) * sms * warps_per_sm * 32);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    dp<MODE, ILP><<<sms * warps_per_sm, 32>>>(out, 1.f);
    cudaEventRecord(a);
    dp<MODE, ILP><<<sms * warps_per_sm, 32>>>(out, 1.f);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    // cells: MODE 0: ILP chains x WCELLS; MODE 1: ILP pairs x WCELLS cells (WCELLS/2 per half x 2)
    const double cells = (double)sms * warps_per_sm * 32 * REPS * ILP * WCELLS;
    printf("%-7s ILP=%d warps/SM=%2d : %7.0f GCUPS\n", MODE ? "packed" : "scalar", ILP, warps_per_sm,
           cells / (ms * 1e-3) / 1e9);
    cudaFree(out);
}

int main() {
    for (int w : {4, 8, 12, 16, 24, 32}) { run<0, 1>(w); run<1, 1>(w); }
    for (int w : {8, 12, 16}) { run<0, 2>(w); run<1, 2>(w); }
    for (int w : {8, 16}) { run<0, 4>(w); run<1, 4>(w); }
    return 0;
}
