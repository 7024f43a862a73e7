// dp_common.cuh -- types shared by the K-DP / K-BT kernels (dp.cu, dp_batch.cu, backtrack.cu).
#pragma once
#include <cstdio>
#include "hgm_device.cuh"
#include "hgm_internal.cuh"

namespace hgm {

// Device-side bounds checks of the shared-memory and history indices (built with
// -DHGM_DEBUG_CHECKS: tests/test_gpu_debug_checks.py).  compute-sanitizer is closed on this
// pool, so the kernels check their own indices: a failed check prints and traps (the call
// then returns HGM_ERR_CUDA).
#ifdef HGM_DEBUG_CHECKS
#define HGM_DCHECK(cond)                                                                                    \
    do {                                                                                                    \
        if (!(cond)) {                                                                                      \
            printf("HGM_DCHECK failed %s:%d block %d thread %d: %s\n", __FILE__, __LINE__, (int)blockIdx.x, \
                   (int)threadIdx.x, #cond);                                                                \
            __trap();                                                                                       \
        }                                                                                                   \
    } while (0)
#else
#define HGM_DCHECK(cond) \
    do {                 \
    } while (0)
#endif

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
    const int32_t *__restrict__ prow_pad;  // row of each padded entry, -1 = padding slot
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
    int32_t ppad;     // padded band index of the window's first row = qpad[wb]
    int32_t npp;      // padded pair slots of the window = qpad[we] - qpad[wb]
    int32_t ntail;    // first dummy-form slot of a layer: np (v0, compact) or npp (padded layout)
    int32_t pad_;
};

// K-DP shared-memory entry of a candidate (b, c_j): the NM messages m^k(b, c_j),
// then theta(b -> c_j), padded to whole float4 (LDS.128) -- dp_batch.cu
__host__ __device__ constexpr int entry_floats(int nm) { return ((nm + 1) + 3) & ~3; }

struct StepConst {
    float g_i, g_im1, A1, K2;  // model gaps (Eq. 5) and angle constants (Eq. 6), hgm_device.cuh
};

struct DPParams {
    float l1, l2, l23, l1W, W;
    int T;
};

// Layer layout of one instance: [pairs | (b,eps) Sw | (eps,a) Sw | (eps,eps) 1], the
// pairs compact (np slots, v0 kernels) or in padded band order (npp slots: state
// (b, a) at qpad[a] - ppad + column of b in row a), model index fastest.
__device__ __forceinline__ int ns_of(const InstDesc &d) { return d.ntail + 2 * (d.we - d.wb) + 1; }

struct TileCaps {  // shared-memory capacities of one K-DP work item, maxima over the call's tiles
    int NE;     // candidate entries (padded band slots of the tile's b rows)
    int TH;     // floats of the padded direction rows [A0, B1) incl. alignment slack
    int NA;     // row-table rows: the a rows before B0 plus the b rows
    int NB;     // b nodes
    int NC;     // candidate nodes [B0, Cend)
    int NST;    // real states
    int FT;     // b-frames
    int W;      // window length in frames
    int STAGE;  // bytes of one K-DP shared-memory stage (largest item layout)
    int NSTAGE; // stages: 2 (the next item streams in while one is processed) or 1 (huge items)
};

// One K-DP work item: a tile of b-frames [F0, F1) of one window (dp_batch.cu).
struct WorkItem {
    InstDesc d;    // the window
    int live;      // 0: end-of-work marker
    int idx;       // index in the chunk's item list (its bookkeeping record)
    int F0, F1;
    int B0, B1;    // b nodes: minnode(F0), minnode(F1)
    int A0;        // first direction row: max(minnode(F0 - T + 1), window start)
    int Cend;      // candidate nodes end: min(minnode(F1 + T - 1), window end)
    int qa, qb0, qb1;  // qpad[A0], qpad[B0], qpad[B1]
    int G0, G1;    // a-frames [G0, G1) of the item's real states (the whole range unless T is large)
    int qa1;       // qpad[minnode(G1)]: end of the direction rows the loop reads
    int primary;   // 1: this item also finishes the b rows' dummy-form states (one item per b-tile)
    int nA;        // row tables: the a rows [A0, A0 + nA) = [A0, min(minnode(G1), B0)), then the b rows
                   // [B0, B1) (large T: an a-frame chunk far before its b-frame needs no rows between)
    // filled by the producer lane: shared-memory index of each range's first element
    int th0, tb0, we0, eb0, ee0, uc0, tc0, rf0, ft0, flo;
};

constexpr int MAX_BATCH = 8;  // models of equal M evaluated together by one CTA

// Batched layouts (NM models of equal M, model index k fastest):
//   unary    U[((i * nn) + (n - n_lo)) * NM + k]
//   history  hist[layer * L + off + s * SS + k]   (SS = entry_floats(NM) floats per state; v0: SS = 1)
// K-DPW (dp_window.cu): per-window kernel, the whole recursion of one window in one CTA.
// Entry width: NM messages + theta(b -> c), float2 for one model, whole float4s otherwise.
__host__ __device__ constexpr int went_floats(int nm) { return nm == 1 ? 2 : entry_floats(nm); }
struct WinCaps {  // maxima over the windows of one launch
    int NPP;      // padded band slots of a window
    int SW;       // window nodes
    int W;        // window length in frames
    int NTASK;    // task capacity (>= the tasks of every window)
    int T;
    int M;        // chain length (the step constants of every step live in shared memory)
};
struct WinStepPtrs {
    const float4 *step[MAX_BATCH];  // per-model step constants (g_i, g_{i-1}, A1, K2), device
};

struct BTArgs {
    const float *U;   // raw U (the appearance distance A)
    const float *Us;  // lambda1 U (the recursion's values)
    int64_t nn, n_lo;
    int NM, M;
    int SS;  // floats per state in a layer (entry_floats(NM); the model index k is slot k)
    const float4 *step[MAX_BATCH];  // per-model step constants (device)
    float *E[MAX_BATCH], *A[MAX_BATCH];
    int64_t *z[MAX_BATCH];  // [count * M] per model
};

struct StepConstB {  // per-model constants of one step, in the kernel parameter space
    float4 c[MAX_BATCH];  // (g_i, g_{i-1}, A1, K2)
    // the same angle constants negated and paired for the packed (f32x2) candidate body:
    // nA1[q] = (-A1_{2q}, -A1_{2q+1}), nK2[q] = (-K2_{2q}, -K2_{2q+1}) (odd batch: last pair repeats)
    float2 nA1[MAX_BATCH / 2], nK2[MAX_BATCH / 2];
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
