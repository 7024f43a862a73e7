// dp_common.cuh -- types shared by the K-DP / K-BT kernels (dp.cu, dp_tiled.cu).
#pragma once
#include "hgm_device.cuh"
#include "hgm_internal.cuh"

namespace hgm {

struct SceneView {
    const int32_t *__restrict__ t;
    const int32_t *__restrict__ ft;
    const int32_t *__restrict__ qstart;
    const float *__restrict__ theta;
    const uint8_t *__restrict__ coinc;
    const uint16_t *__restrict__ cpre;  // per-row inclusive prefix count of coinc
    const int32_t *__restrict__ prow;
    const int64_t *__restrict__ id;
    const int32_t *__restrict__ qpad;      // padded band (K-DP staging)
    const float *__restrict__ theta_pad;
    const int32_t *__restrict__ rfc, *__restrict__ rlc;  // per-row first / last coincident column
    const int4 *__restrict__ ninfo;  // (t', minnode(t'+1), qstart, qpad) per node
    int fmax, S;
    __device__ __forceinline__ int first(int f) const { return first_at(ft, fmax, S, f); }
    // coincident pairs in row x, columns [j0, j1)
    __device__ __forceinline__ int coinc_count(int q, int j0, int j1) const {
        if (j1 <= j0) return 0;
        return (int)__ldg(cpre + q + j1 - 1) - (j0 > 0 ? (int)__ldg(cpre + q + j0 - 1) : 0);
    }
};

struct InstDesc {
    int32_t wb, we;   // window node range [wb, we)
    int32_t pbase;    // band index of the window's first row = qstart[wb]
    int32_t np;       // pair states of the window = qstart[we] - qstart[wb]
    int64_t off;      // offset of this instance inside a layer
    int32_t out;      // output slot (offset index)
    int32_t o;        // first frame of the window
    int64_t moff;     // offset of this instance's message rows in the message buffer (floats)
    int32_t ppad;     // padded band index of the window's first row = qpad[wb]
    int32_t pad_;
};

// Message buffer layout (per instance, padded band order, model index fastest):
//   msg[moff + (qpad[b] - ppad + j) * nm_pad(NM) + k] = m^k_i(b, c_j)
// element stride of the message rows: aligned for LDS.64 / LDS.128 vector loads
__host__ __device__ constexpr int nm_pad(int nm) {
    return nm <= 1 ? 1 : nm <= 2 ? 2 : nm <= 4 ? 4 : nm <= 6 ? 6 : 8;
}

struct StepConst {
    float g_i, g_im1, A1, K2;  // model gaps (Eq. 5) and angle constants (Eq. 6), hgm_device.cuh
};

struct DPParams {
    float l1, l2, l23, l1W, W;
    int T;
};

// Layer layout of one instance: [pairs np | (b,eps) Sw | (eps,a) Sw | (eps,eps) 1]
__device__ __forceinline__ int ns_of(const InstDesc &d) { return d.np + 2 * (d.we - d.wb) + 1; }

struct TileGeom {  // shared-memory capacities of one K-DP tile, upper bounds over the call
    int FT;     // b-frames per tile
    int NB;     // message rows (b nodes) per tile
    int NA;     // direction rows (a and b nodes) per tile
    int TH;     // floats of the padded direction rows
    int MT;     // float2 of the padded message rows
    int NST;    // real states per tile
    int W;      // window length in frames
    int ntile;  // tiles per window
};

constexpr int MAX_BATCH = 8;  // models of equal M evaluated together by one CTA

// Batched layouts (NM models of equal M, model index k fastest):
//   unary    U[((i * nn) + (n - n_lo)) * NM + k]
//   history  hist[layer * L + off + s * NM + k]   (off counts states x NM)
struct BTArgs {
    const float *U;
    int64_t nn, n_lo;
    int NM, M;
    const float4 *step[MAX_BATCH];  // per-model step constants (device)
    float *E[MAX_BATCH], *A[MAX_BATCH];
    int64_t *z[MAX_BATCH];  // [count * M] per model
};

struct StepConstB {  // per-model constants of one step, in the kernel parameter space
    float4 c[MAX_BATCH];  // (g_i, g_{i-1}, A1, K2)
};

__device__ __forceinline__ float warp_min(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

__device__ __forceinline__ float min3(float a, float b, float c) {
    float r;
    asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}

}  // namespace hgm
