// msg.cu -- K-MSG: hoisted messages and dummy-form states of one recursion step
// for a batch of NM models (streaming kernel, one thread per band entry).
//
// For step i (Eq. 10) and every real pair (x -> c) of the window
// (c in frames (t'(x), t'(x)+T)):
//   n^k(x,c) = alpha^k_{i+1}(c, x) + lambda1 U^k_i(c)
//   m^k(x,c) = n^k(x,c) + lambda2 |g^k_i - (t'(c) - t'(x))|        -> message buffer
// and the states whose recursion has no geometric term (reading R5):
//   alpha_i(x, eps)   = min( min_c n(x,c),  lambda1 W^d + alpha_{i+1}(eps, x) )
//   alpha_i(eps, x)   = min( min_c w(c),    lambda1 W^d + alpha_{i+1}(eps, eps) )
//   alpha_i(eps, eps) = min( min_{c in window} w(c), lambda1 W^d + alpha_{i+1}(eps, eps) )
// with w(c) = alpha_{i+1}(c, eps) + lambda1 U_i(c).
//
// Layout for bandwidth: CTAs 1.. of a window take one band entry per thread
// (rows are contiguous in the compact alpha layer and in the padded message
// buffer, so loads and stores coalesce); the (x, eps) row minimum is one
// match_any + one redux.sync per model over the lanes of the same row, finished
// by one atomicMin per row run and model on the row's slot (non-negative floats
// order like their bits).  That slot holds the dummy term lambda1 W^d +
// alpha_{i+1}(eps, x) beforehand: K-INIT for the first step of a chunk, the
// previous K-DP launch for the others (dp_batch.cu).  CTA 0 of a window does the
// per-node part: w(c), per-frame minima, then (eps, x) and (eps, eps) directly.
// The arithmetic is hgm_device.cuh's, so K-BT's re-evaluation stays bit-identical.
#include <algorithm>

#include "dp_common.cuh"

namespace hgm {

constexpr int KM_THREADS = 256;
constexpr int KM_PER_THREAD = 4;  // band entries per thread (contiguous across the CTA)

template <int NM>
__device__ __forceinline__ void ld_vec(const float *__restrict__ src, float (&v)[NM]) {
    if constexpr (NM % 2 == 0) {
#pragma unroll
        for (int q = 0; q < NM / 2; ++q) {
            const float2 t = __ldg(reinterpret_cast<const float2 *>(src) + q);
            v[2 * q] = t.x;
            v[2 * q + 1] = t.y;
        }
    } else {
#pragma unroll
        for (int q = 0; q < NM; ++q) v[q] = __ldg(src + q);
    }
}

constexpr int KM_MAXW = 512;  // window frames handled by the per-node pass (larger windows: global fallback)

template <int NM, bool kHasNext>
__global__ void __launch_bounds__(KM_THREADS) k_msg(SceneView sc, const InstDesc *__restrict__ inst,
                                                    float *__restrict__ hist, int64_t L, int layer, StepConstB kc,
                                                    const float *__restrict__ Ui, float *__restrict__ msg, DPParams p,
                                                    int W) {
    constexpr int NMP = nm_pad(NM);
    const InstDesc d = inst[blockIdx.y];
    const int lane = threadIdx.x & 31;
    const int Sw = d.we - d.wb;
    float *cur = hist + (int64_t)layer * L + d.off;
    const float *nxt = kHasNext ? hist + (int64_t)(layer + 1) * L + d.off : nullptr;
    if (blockIdx.x == 0) {
        // ---- per-node pass: w(c) = alpha_{i+1}(c, eps) + lambda1 U_i(c); frame minima; (eps, x) and (eps, eps)
        __shared__ float s_fm[KM_MAXW * NM];
        const bool fits = W <= KM_MAXW;
        if (fits) {
            for (int q = threadIdx.x; q < W * NM; q += KM_THREADS) {
                const int fi = q / NM, k = q - fi * NM, f = d.o + fi;
                const int c1 = min(sc.first(f + 1), d.we);
                float w = INFINITY;
                for (int c = sc.first(f); c < c1; ++c)
                    w = fminf(w, msg_n(kHasNext ? nxt[(int64_t)(d.np + (c - d.wb)) * NM + k] : 0.f, p.l1,
                                       __ldg(Ui + (int64_t)c * NM + k)));
                s_fm[q] = w;
            }
        }
        __syncthreads();
        for (int q = threadIdx.x; q < (Sw + 1) * NM; q += KM_THREADS) {
            const int xi = q / NM, k = q - xi * NM;
            const float ee_next = kHasNext ? nxt[(int64_t)(d.np + 2 * Sw) * NM + k] : 0.f;
            float r = INFINITY;
            int f0, f1;
            if (xi < Sw) {  // (eps, x): candidates in frames (t'(x), t'(x)+T) inside the window
                const int tx = sc.t[d.wb + xi];
                f0 = tx + 1;
                f1 = min(tx + p.T, d.o + W);
            } else {  // (eps, eps): the whole window
                f0 = d.o;
                f1 = d.o + W;
            }
            if (fits) {
                for (int f = f0; f < f1; ++f) r = fminf(r, s_fm[(f - d.o) * NM + k]);
            } else {
                const int c1 = min(sc.first(f1), d.we);
                for (int c = sc.first(f0); c < c1; ++c)
                    r = fminf(r, msg_n(kHasNext ? nxt[(int64_t)(d.np + (c - d.wb)) * NM + k] : 0.f, p.l1,
                                       __ldg(Ui + (int64_t)c * NM + k)));
            }
            cur[(int64_t)(d.np + Sw + xi) * NM + k] = fminf(r, __fadd_rn(p.l1W, ee_next));
        }
        return;
    }
    // ---- band entries: messages and the (x, eps) row minima
    unsigned *slot_be = reinterpret_cast<unsigned *>(cur + (int64_t)d.np * NM);
    const int64_t base =
        (int64_t)(blockIdx.x - 1) * (KM_THREADS * KM_PER_THREAD) + (threadIdx.x & ~31) * KM_PER_THREAD;
#pragma unroll
    for (int u = 0; u < KM_PER_THREAD; ++u) {
        const int64_t le = base + u * 32 + lane;  // local band entry of the window
        const bool inr = le < d.np;
        int x = -1, c = 0, j = 0, dt = 0;
        int4 ni = make_int4(0, 0, 0, 0);
        if (inr) {
            x = __ldg(sc.prow + d.pbase + le);
            ni = __ldg(sc.ninfo + x);  // (t'(x), minnode(t'(x)+1), qstart, qpad)
            j = (int)(d.pbase + le - ni.z);
            c = ni.y + j;
            if (c < d.we) dt = __ldg(sc.t + c) - ni.x;
        }
        // the band row may run past the window, and the band is built for T_max >= T
        const bool ok = inr && c < d.we && dt < p.T;
        float n[NM];
#pragma unroll
        for (int k = 0; k < NM; ++k) n[k] = INFINITY;
        if (ok) {
            float a[NM], uu[NM];
            if (kHasNext) ld_vec<NM>(nxt + le * NM, a);
            ld_vec<NM>(Ui + (int64_t)c * NM, uu);
            float m[NMP];
#pragma unroll
            for (int k = 0; k < NM; ++k) {
                n[k] = msg_n(kHasNext ? a[k] : 0.f, p.l1, uu[k]);
                m[k] = msg_m(n[k], p.l2, kc.c[k].x, dt);
            }
            float *dst = msg + d.moff + (int64_t)(ni.w - d.ppad + j) * NMP;
            if constexpr (NM % 2 == 0) {
#pragma unroll
                for (int q = 0; q < NM / 2; ++q) reinterpret_cast<float2 *>(dst)[q] = make_float2(m[2 * q], m[2 * q + 1]);
            } else {
#pragma unroll
                for (int k = 0; k < NM; ++k) dst[k] = m[k];
            }
        }
        // per-row minima: one pass per distinct row in the warp (rows are contiguous lane
        // runs, typically 2 per warp); full-warp redux.sync on masked values (a redux with
        // a partial mask serialises), one atomic per row run and model
        unsigned todo = __ballot_sync(0xffffffffu, ok);
        while (todo) {
            const int src = __ffs(todo) - 1;
            const int r = __shfl_sync(0xffffffffu, x, src);
            const bool mine = ok && x == r;
            todo &= ~__ballot_sync(0xffffffffu, mine);
#pragma unroll
            for (int k = 0; k < NM; ++k) {
                const unsigned v = __reduce_min_sync(0xffffffffu, mine ? __float_as_uint(n[k]) : 0x7f800000u);
                if (lane == src) atomicMin(slot_be + (int64_t)(r - d.wb) * NM + k, v);
            }
        }
    }
}

// K-INIT: dummy term of the first step's (x, eps) slots (alpha_{M+1} = 0)
template <int NM>
__global__ void k_msg_init(const InstDesc *__restrict__ inst, float *__restrict__ hist, int64_t L, int layer,
                           float l1W) {
    const InstDesc d = inst[blockIdx.y];
    const int Sw = d.we - d.wb;
    float *cur = hist + (int64_t)layer * L + d.off;
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < Sw * NM; q += gridDim.x * blockDim.x)
        cur[(int64_t)d.np * NM + q] = __fadd_rn(l1W, 0.f);
}

template <int NM>
static void launch_msg_nm(const SceneView &v, const InstDesc *dinst, int ninst, int max_np, int max_sw, float *hist,
                          int64_t L, int layer, bool has_next, bool init, const StepConstB &kc, const float *Ui,
                          float *msg, const DPParams &p, int W, cudaStream_t s) {
    if (init) {
        const dim3 gi((unsigned)std::max(1, (max_sw * NM + 255) / 256), (unsigned)ninst);
        k_msg_init<NM><<<gi, 256, 0, s>>>(dinst, hist, L, layer, p.l1W);
    }
    const int per_cta = KM_THREADS * KM_PER_THREAD;
    const dim3 grid((unsigned)(1 + std::max(1, (max_np + per_cta - 1) / per_cta)), (unsigned)ninst);
    if (has_next) k_msg<NM, true><<<grid, KM_THREADS, 0, s>>>(v, dinst, hist, L, layer, kc, Ui, msg, p, W);
    else k_msg<NM, false><<<grid, KM_THREADS, 0, s>>>(v, dinst, hist, L, layer, kc, Ui, msg, p, W);
}

hgm_status launch_msg(int NM, const SceneView &v, const InstDesc *dinst, int ninst, int max_np, int max_sw,
                      float *hist, int64_t L, int layer, bool has_next, bool init, const StepConstB &kc,
                      const float *Ui, float *msg, const DPParams &p, int W, cudaStream_t s) {
#define HGM_NM_CASE(n) \
    case n: launch_msg_nm<n>(v, dinst, ninst, max_np, max_sw, hist, L, layer, has_next, init, kc, Ui, msg, p, W, s); break
    switch (NM) {
        HGM_NM_CASE(1);
        HGM_NM_CASE(2);
        HGM_NM_CASE(3);
        HGM_NM_CASE(4);
        HGM_NM_CASE(5);
        HGM_NM_CASE(6);
        HGM_NM_CASE(7);
        HGM_NM_CASE(8);
        default: return fail(HGM_ERR_INVALID_ARGUMENT, "model batch size must be 1..8");
    }
#undef HGM_NM_CASE
    return HGM_OK;
}

}  // namespace hgm
