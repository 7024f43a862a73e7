// unary.cu -- K-U: the unary look-up table of PAPER.md §3.3 (L341-366).
//
//   U[j][n] = || f_j - f'_n ||_2   (Eq. 2)
//
// for every model node j of the call (all models concatenated) and every scene
// node n of the covered range.  Direct differences with four partial sums in
// fp32 and a correctly rounded square root.  The GEMM expansion
// |f|^2 + |f'|^2 - 2 f.f' is NOT used: it cancels for near matches (U ~ 0)
// and would miss the 1e-6 absolute tolerance, which is also
// why this is not a tensor-core contraction.
//
// Two tables are written: U (the appearance distance A of the backtrack sums it)
// and Us = lambda1 * U rounded once (the recursion's unary term; every K-DP / K-BT kernel
// reads Us, so the product is formed once per (node, scene node) instead of per message).
//
// Layout: a CTA owns a tile of TN scene nodes and loops over model nodes in
// tiles of TJ staged in shared memory; each thread keeps its scene node's
// running partial sums for TJ model nodes in registers while streaming the
// scene descriptor once per model tile (float4, L1-friendly).
#include "hgm_device.cuh"
#include "hgm_internal.cuh"

namespace hgm {

constexpr int KU_TN = 128;  // scene nodes per CTA (one per thread)
constexpr int KU_TJ = 8;    // model nodes per register tile

__global__ void __launch_bounds__(KU_TN) k_unary(ModelFeats mf, int M, int NM, int Fp,
                                                 const float *__restrict__ sfeat, int64_t n_lo, int64_t nn,
                                                 int tiles_per_y, float l1, float *__restrict__ U,
                                                 float *__restrict__ Us) {
    const int M_total = M * NM;
    // blockIdx.y owns model-node tiles [y * tiles_per_y, (y + 1) * tiles_per_y): small
    // scenes (few scene tiles) still fill the GPU
    const int j_begin = blockIdx.y * tiles_per_y * KU_TJ, j_end = min(M_total, j_begin + tiles_per_y * KU_TJ);
    extern __shared__ float4 sm[];  // [KU_TJ][Fp/4] model descriptors
    const int F4 = Fp >> 2;
    const int64_t n = blockIdx.x * (int64_t)KU_TN + threadIdx.x;
    const bool live = n < nn;
    const float4 *srow = reinterpret_cast<const float4 *>(sfeat + (n_lo + (live ? n : 0)) * (int64_t)Fp);
    for (int j0 = j_begin; j0 < j_end; j0 += KU_TJ) {
        const int nj = min(KU_TJ, j_end - j0);
        __syncthreads();
        for (int k = threadIdx.x; k < nj * F4; k += KU_TN) {  // node j = model kk's node i, read in place
            const int q = k / F4, r = k - q * F4, j = j0 + q, kk = j / M, i = j - kk * M;
            sm[k] = reinterpret_cast<const float4 *>(mf.p[kk] + (int64_t)i * Fp)[r];
        }
        __syncthreads();
        float acc[KU_TJ][4];
#pragma unroll
        for (int q = 0; q < KU_TJ; ++q) acc[q][0] = acc[q][1] = acc[q][2] = acc[q][3] = 0.f;
        // unrolled so that several scene-descriptor loads are in flight (a small scene
        // launches few CTAs and each thread's loop is otherwise one load latency per float4);
        // every accumulator still sums its k in order, so the table's bits do not change
#pragma unroll 4
        for (int k = 0; k < F4; ++k) {
            const float4 v = __ldg(srow + k);
#pragma unroll
            for (int q = 0; q < KU_TJ; ++q) {
                if (q < nj) {
                    const float4 u = sm[q * F4 + k];
                    float d0 = __fsub_rn(u.x, v.x), d1 = __fsub_rn(u.y, v.y);
                    float d2 = __fsub_rn(u.z, v.z), d3 = __fsub_rn(u.w, v.w);
                    acc[q][0] = __fmaf_rn(d0, d0, acc[q][0]);
                    acc[q][1] = __fmaf_rn(d1, d1, acc[q][1]);
                    acc[q][2] = __fmaf_rn(d2, d2, acc[q][2]);
                    acc[q][3] = __fmaf_rn(d3, d3, acc[q][3]);
                }
            }
        }
        if (live) {
#pragma unroll
            for (int q = 0; q < KU_TJ; ++q)
                if (q < nj) {
                    const int j = j0 + q, k = j / M, i = j - k * M;  // node j = k*M + i of model k
                    const float u =
                        __fsqrt_rn(__fadd_rn(__fadd_rn(acc[q][0], acc[q][1]), __fadd_rn(acc[q][2], acc[q][3])));
                    U[((int64_t)i * nn + n) * NM + k] = u;
                    Us[((int64_t)i * nn + n) * NM + k] = scale_l1(l1, u);  // the recursion's lambda1 U
                }
        }
    }
}

hgm_status unary_table(const ModelFeats &mf, int M, int NM, int Fp, const hgm_scene *sc, int64_t n_lo, int64_t n_hi,
                       float l1, float *U, float *Us, cudaStream_t s) {
    const int64_t nn = n_hi - n_lo;
    if (nn <= 0 || M * NM <= 0) return HGM_OK;
    Timer tm(s, K_UNARY);
    const size_t smem = sizeof(float) * KU_TJ * Fp;
    if (smem > 48 * 1024) HGM_CUDA(cudaFuncSetAttribute(k_unary, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int64_t gx = (nn + KU_TN - 1) / KU_TN;
    const int jt = (M * NM + KU_TJ - 1) / KU_TJ;                              // model-node tiles
    const int gy_want = (int)std::min<int64_t>(jt, std::max<int64_t>(1, (4 * 148 + gx - 1) / gx));
    const int tpy = (jt + gy_want - 1) / gy_want, gy = (jt + tpy - 1) / tpy;
    k_unary<<<dim3((unsigned)gx, (unsigned)gy), KU_TN, smem, s>>>(mf, M, NM, Fp, sc->feat, n_lo, nn, tpy, l1, U, Us);
    count_launch(K_UNARY);
    HGM_CUDA(cudaGetLastError());
    return HGM_OK;
}

}  // namespace hgm
