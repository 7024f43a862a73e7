// pipe_microbench.cu -- issue/pipe throughput of the instructions the K-DP candidate
// loop is made of, measured on the box (DESIGN.md §6 roofline): FADD, FFMA, FFMA2/FADD2
// (packed f32x2, sm_100), MUFU.SQRT (sqrt.approx.ftz), FMNMX3 (3-input min).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pmb tools/pipe_microbench.cu
#include <cstdio>
#include <cuda_runtime.h>

#define N_IT 4096
typedef unsigned long long u64;

__device__ __forceinline__ u64 ffma2(u64 a, u64 b, u64 c) { u64 r; asm volatile("fma.rn.f32x2 %0,%1,%2,%3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r; }
__device__ __forceinline__ float sq(float x) { float r; asm volatile("sqrt.approx.ftz.f32 %0,%1;" : "=f"(r) : "f"(x)); return r; }
__device__ __forceinline__ float mn3(float a, float b, float c) { float r; asm volatile("min.f32 %0,%1,%2,%3;" : "=f"(r) : "f"(a), "f"(b), "f"(c)); return r; }

template <int KIND>
__global__ void k(float *out, float s) {
    float a[8];
    u64 p[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) { a[u] = s * (threadIdx.x + u); p[u] = (u64)__float_as_uint(a[u]) | ((u64)__float_as_uint(a[u] + 1.f) << 32); }
    const u64 m = (u64)__float_as_uint(0.999f) | ((u64)__float_as_uint(0.998f) << 32);
    const u64 c = (u64)__float_as_uint(0.001f) | ((u64)__float_as_uint(0.002f) << 32);
    for (int it = 0; it < N_IT; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            if (KIND == 0) asm volatile("fma.rn.f32 %0,%0,%1,%2;" : "+f"(a[u]) : "f"(0.999f), "f"(0.001f));
            if (KIND == 1) p[u] = ffma2(p[u], m, c);
            if (KIND == 2) a[u] = sq(a[u] + 1.0f);   // MUFU + FADD
            if (KIND == 3) a[u] = mn3(a[u], a[(u + 1) & 7], 5.f);
            if (KIND == 4) { a[u] = sq(a[u]); }   // MUFU alone (dependent chain per u)
        }
    }
    float r = 0;
#pragma unroll
    for (int u = 0; u < 8; ++u) r += a[u] + __uint_as_float((unsigned)p[u]);
    if (r == 12345.f) out[0] = r;
}

int main() {
    float *d; cudaMalloc(&d, 4);
    int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const char *names[] = {"FFMA", "FFMA2 (f32x2)", "MUFU.SQRT+FADD", "FMNMX3", "MUFU.SQRT"};
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int kind = 0; kind < 5; ++kind) {
        for (int rep = 0; rep < 2; ++rep) {
            const int blocks = nsm * 4, threads = 512;
            cudaEventRecord(e0);
            switch (kind) {
                case 0: k<0><<<blocks, threads>>>(d, 1e-3f); break;
                case 1: k<1><<<blocks, threads>>>(d, 1e-3f); break;
                case 2: k<2><<<blocks, threads>>>(d, 1e-3f); break;
                case 3: k<3><<<blocks, threads>>>(d, 1e-3f); break;
                case 4: k<4><<<blocks, threads>>>(d, 1e-3f); break;
            }
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            const double warp_inst = (double)blocks * threads / 32 * N_IT * 8;
            if (rep) printf("%-16s %8.3f ms  %.3f warp-inst/clk/SM (at %d MHz nominal; %.1f G warp-inst/s)\n", names[kind], ms,
                            warp_inst / (ms * 1e-3) / nsm / (clk * 1e3), clk / 1000, warp_inst / (ms * 1e-3) / 1e9);
        }
    }
    return 0;
}
