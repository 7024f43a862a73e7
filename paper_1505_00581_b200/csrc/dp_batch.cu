// dp_batch.cu -- K-DP: the real states of one recursion step (Eq. 10)
// for a batch of NM models of equal chain length M against one window, one CTA
// per (window, tile of FT consecutive b-frames), one launch per step i.
//
//   alpha^k_i(b, a) = min( min_{c in L(b,a)} [ m^k(b,c) + lambda2 lambda3 Dg^k(c,b,a) ]
//                          + lambda2 |g^k_{i-1} - (t'(b) - t'(a))|,
//                          lambda1 W^d + alpha^k_{i+1}(eps, b) )
// with L(b,a) = [minnode(t'(b)+1), minnode(t'(a)+T)) (R1-R3)
// and the hoisted messages m written by K-MSG (msg.cu).
//
// Everything that depends only on the scene is shared by the NM models: the
// direction rows, the state set and its decode, and the two scene-angle folds
// of every candidate (hgm_device.cuh).  Per model and candidate only
// e1 = fold_b - A1, e2 = fold_c - K2, e1^2 + e2^2, one MUFU.SQRT, the FFMA onto
// the message and the min remain (~6.5 issue slots instead of 10.5).
//
// Phase 0  two cp.async range copies (direction rows x in [A0, B1) from the
//          padded band, message rows b in [B0, B1) from the message buffer; odd
//          padded row lengths put consecutive rows on distinct banks), row
//          bookkeeping (one int4 per node), the segment table of the real states
//          (a (b-frame, a-frame) segment shares its candidate range), and the
//          dummy terms of the NEXT layer's (b, eps), (eps, b) slots for the
//          tile's b nodes (K-MSG of step i-1 min-reduces into them).
// Phase 1  segment prefix + state -> segment map (one warp).
// Phase 2  real states, one per lane, ordered by frame gap, so the lanes of a
//          warp see near-equal trip counts.  States touching a coincident pair
//          (R10) take the exact flag-aware loop.
#include "dp_common.cuh"

namespace hgm {

struct Seg {  // one (b-frame f, a-frame f-g) block of real states
    int start;     // first state index (prefix over segments)
    int b0, nb;    // b nodes [b0, b0+nb): frame f
    int a0;        // a nodes start: frame f-g
    int trip;      // candidates per state
    int aoff;      // column of the first candidate in the rows of frame f-g
    int f1a;       // minnode(f-g+1): column origin of the rows of frame f-g
    int g;         // frame gap t'(b) - t'(a)
    unsigned inv;  // ceil(2^32 / nb): division-free state decode
};

constexpr int KDP_THREADS = 256;
constexpr int KDP_WARPS = KDP_THREADS / 32;

__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~(size_t)15; }

struct SmemPlan {
    size_t th, mt, rows, brows, seg, map, total;
    __host__ __device__ SmemPlan(const TileGeom &tg, int T, int NM) {
        th = 0;
        mt = align16(th + sizeof(float) * (size_t)tg.TH);
        rows = align16(mt + sizeof(float) * (size_t)nm_pad(NM) * tg.MT);
        brows = align16(rows + sizeof(int) * 5 * (size_t)tg.NA);
        seg = align16(brows + sizeof(float) * (size_t)NM * tg.NB);
        map = align16(seg + sizeof(Seg) * (size_t)tg.FT * (T - 1));
        total = align16(map + (size_t)tg.NST);
    }
};

__device__ __forceinline__ int warp_incl_scan(int v, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
    }
    return v;
}

__device__ __forceinline__ void cp_async16(void *smem_dst, const void *gmem_src) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(gmem_src));
}

// copy floats [g0, g1) of src to dst so that dst[q] holds src[a0 + q], a0 = g0 & ~3; returns a0
__device__ __forceinline__ int64_t copy_range(float *dst, const float *src, int64_t g0, int64_t g1, int tid) {
    const int64_t a0 = g0 & ~(int64_t)3, a1 = (g1 + 3) & ~(int64_t)3;
    for (int64_t q = tid; q < (a1 - a0) >> 2; q += KDP_THREADS) cp_async16(dst + 4 * q, src + a0 + 4 * q);
    return a0;
}

template <int NMP>
__device__ __forceinline__ void load_msgs(const float *__restrict__ src, float (&m)[NMP]) {
    if constexpr (NMP == 6) {
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            const float2 v = reinterpret_cast<const float2 *>(src)[q];
            m[2 * q] = v.x;
            m[2 * q + 1] = v.y;
        }
    } else if constexpr (NMP >= 4) {
#pragma unroll
        for (int q = 0; q < NMP / 4; ++q) {
            const float4 v = reinterpret_cast<const float4 *>(src)[q];
            m[4 * q] = v.x;
            m[4 * q + 1] = v.y;
            m[4 * q + 2] = v.z;
            m[4 * q + 3] = v.w;
        }
    } else if constexpr (NMP == 2) {
        const float2 v = *reinterpret_cast<const float2 *>(src);
        m[0] = v.x;
        m[1] = v.y;
    } else {
        m[0] = *src;
    }
}

template <int NM>
__device__ __forceinline__ void store_msgs(float *__restrict__ dst, const float (&v)[NM]) {
    if constexpr (NM % 2 == 0) {
#pragma unroll
        for (int q = 0; q < NM / 2; ++q) reinterpret_cast<float2 *>(dst)[q] = make_float2(v[2 * q], v[2 * q + 1]);
    } else {
#pragma unroll
        for (int q = 0; q < NM; ++q) dst[q] = v[q];
    }
}

template <int NM, bool kHasNext>
__global__ void __launch_bounds__(KDP_THREADS) k_dp_batch(SceneView sc, const InstDesc *__restrict__ inst,
                                                          float *__restrict__ hist, int64_t L, int layer, int has_prev,
                                                          StepConstB kc, const float *__restrict__ msg, DPParams p,
                                                          TileGeom tg) {
    constexpr int NMP = nm_pad(NM);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const SmemPlan sp(tg, p.T, NM);
    float *TH = reinterpret_cast<float *>(smem_raw + sp.th);
    float *MT = reinterpret_cast<float *>(smem_raw + sp.mt);
    int *r_ofs = reinterpret_cast<int *>(smem_raw + sp.rows);  // [NA] offset of row x in TH
    int *r_q = r_ofs + tg.NA;                                     // qstart[x] (compact band: state index)
    int *r_mo = r_q + tg.NA;                                      // offset of row x in MT (b rows)
    int *r_fc = r_mo + tg.NA;                                     // first / last coincident column
    int *r_lc = r_fc + tg.NA;
    float *b_ean = reinterpret_cast<float *>(smem_raw + sp.brows);  // [NB][NM] alpha_{i+1}(eps, b)
    Seg *seg = reinterpret_cast<Seg *>(smem_raw + sp.seg);
    uint8_t *smap = smem_raw + sp.map;
    __shared__ int s_nst;

    const InstDesc d = inst[blockIdx.y];
    const int T = p.T;
    const int F0 = d.o + blockIdx.x * tg.FT;
    const int wend = d.o + tg.W;
    if (F0 >= wend) return;
    const int F1 = min(F0 + tg.FT, wend);
    const int B0 = sc.first(F0), B1 = sc.first(F1);
    const int A0 = max(sc.first(F0 - T + 1), d.wb);
    const int NR = B1 - A0, NBr = B1 - B0;
    const int Sw = d.we - d.wb;
    float *cur = hist + (int64_t)layer * L + d.off;
    const float *nxt = kHasNext ? hist + (int64_t)(layer + 1) * L + d.off : nullptr;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nseg = tg.FT * (T - 1);

    // ---------------- phase 0
    int64_t th0 = 0, mt0 = 0;  // source index held by TH[0] / MT[0]
    if (NR > 0) {
        const int qa = __ldg(sc.qpad + A0), qb0 = __ldg(sc.qpad + B0), qb1 = __ldg(sc.qpad + B1);
        th0 = copy_range(TH, sc.theta_pad, qa, qb1, tid);
        if (NBr > 0)
            mt0 = copy_range(MT, msg + d.moff, (int64_t)(qb0 - d.ppad) * NMP, (int64_t)(qb1 - d.ppad) * NMP, tid);
        asm volatile("cp.async.commit_group;");
    }
    for (int r = tid; r < NR; r += KDP_THREADS) {
        const int x = A0 + r;
        const int4 ni = __ldg(sc.ninfo + x);  // (t', minnode(t'+1), qstart, qpad)
        r_ofs[r] = (int)(ni.w - th0);
        r_mo[r] = (int)((int64_t)(ni.w - d.ppad) * NMP - mt0);
        r_q[r] = ni.z;
        r_fc[r] = __ldg(sc.rfc + x);  // whole (unclipped) row: conservative
        r_lc[r] = __ldg(sc.rlc + x);
    }
    for (int q = tid; q < NBr * NM; q += KDP_THREADS) {
        const int rb = q / NM, k = q - rb * NM;
        const int64_t sb = (int64_t)(B0 + rb - d.wb);
        b_ean[q] = kHasNext ? nxt[(d.np + Sw + sb) * NM + k] : 0.f;
        if (has_prev)  // dummy term of layer i-1's (b, eps) slot; K-MSG(i-1) min-reduces into it
            (cur - L)[(d.np + sb) * NM + k] = __fadd_rn(p.l1W, cur[(d.np + Sw + sb) * NM + k]);
    }
    for (int s = tid; s < nseg; s += KDP_THREADS) {  // segments, gap-major: long candidate ranges first
        Seg sg{};
        int cnt = 0;
        const int g = 1 + s / tg.FT;
        const int f = F0 + s % tg.FT;
        if (f < F1 && f - g >= d.o) {
            sg.g = g;
            sg.b0 = sc.first(f);
            sg.nb = sc.first(f + 1) - sg.b0;
            sg.a0 = sc.first(f - g);
            sg.f1a = sc.first(f - g + 1);
            const int c0 = sc.first(f + 1);
            sg.trip = max(0, min(sc.first(f - g + T), d.we) - c0);
            sg.aoff = c0 - sg.f1a;
            sg.inv = sg.nb > 1 ? (unsigned)((0x100000000ull + sg.nb - 1) / sg.nb) : 0u;
            cnt = sg.nb * (sg.f1a - sg.a0);
        }
        sg.start = cnt;  // count; prefix below
        seg[s] = sg;
    }
    __syncthreads();
    // ---------------- phase 1: segment prefix + state -> segment map
    if (warp == 0) {
        int carry = 0;
        for (int r0 = 0; r0 < nseg; r0 += 32) {
            const int r = r0 + lane;
            const int v = r < nseg ? seg[r].start : 0;
            const int incl = warp_incl_scan(v, lane);
            if (r < nseg) seg[r].start = carry + incl - v;
            carry += __shfl_sync(0xffffffffu, incl, 31);
        }
        if (lane == 0) s_nst = carry;
    }
    __syncthreads();
    const int nst = s_nst;
    for (int s = warp; s < nseg; s += KDP_WARPS) {
        const int st0 = seg[s].start, cnt = (s + 1 < nseg ? seg[s + 1].start : nst) - st0;
        for (int q = lane; q < cnt; q += 32) smap[st0 + q] = (uint8_t)s;
    }
    asm volatile("cp.async.wait_all;");
    __syncthreads();

    // ---------------- phase 2: real states (b, a)
    for (int s0 = warp * 32; s0 < nst; s0 += KDP_THREADS) {
        const int s = s0 + lane;
        const bool live = s < nst;
        const Seg sg = seg[live ? smap[s] : smap[nst - 1]];
        int trip = 0, b = B0, a = A0;
        if (live) {
            const int r = s - sg.start;
            const int ai = sg.nb > 1 ? (int)__umulhi((unsigned)r, sg.inv) : r;
            b = sg.b0 + (r - ai * sg.nb);
            a = sg.a0 + ai;
            trip = sg.trip;
        }
        const int ra = a - A0, rbt = b - A0;
        const int colb = b - sg.f1a;  // column of b in row a
        const float *mrow = MT + r_mo[rbt];
        const float *brow = TH + r_ofs[rbt];
        const float *arow = TH + r_ofs[ra] + sg.aoff;
        const float th_ab = live ? TH[r_ofs[ra] + colb] : 0.f;
        const int lca = r_lc[ra];
        const bool dirty = live && ((lca >= 0 && lca >= min(colb, sg.aoff) &&
                                     r_fc[ra] <= max(colb, sg.aoff + trip - 1)) || r_fc[rbt] < trip);
        float R[NM];
#pragma unroll
        for (int k = 0; k < NM; ++k) R[k] = INFINITY;
        if (!__any_sync(0xffffffffu, dirty)) {
            int j = 0;
            for (; j + 1 < trip; j += 2) {
                float m0[NMP], m1[NMP];
                load_msgs<NMP>(mrow + (size_t)j * NMP, m0);
                load_msgs<NMP>(mrow + (size_t)(j + 1) * NMP, m1);
                const float b0 = brow[j], b1 = brow[j + 1];
                const float fb0 = fold(b0, th_ab), fc0 = fold(b0, arow[j]);
                const float fb1 = fold(b1, th_ab), fc1 = fold(b1, arow[j + 1]);
#pragma unroll
                for (int k = 0; k < NM; ++k) {
                    const float v0 = __fmaf_rn(p.l23, dg_norm(fb0, fc0, kc.c[k].z, kc.c[k].w), m0[k]);
                    const float v1 = __fmaf_rn(p.l23, dg_norm(fb1, fc1, kc.c[k].z, kc.c[k].w), m1[k]);
                    R[k] = min3(R[k], v0, v1);
                }
            }
            if (j < trip) {
                float m0[NMP];
                load_msgs<NMP>(mrow + (size_t)j * NMP, m0);
                const float b0 = brow[j];
                const float fb0 = fold(b0, th_ab), fc0 = fold(b0, arow[j]);
#pragma unroll
                for (int k = 0; k < NM; ++k)
                    R[k] = fminf(R[k], __fmaf_rn(p.l23, dg_norm(fb0, fc0, kc.c[k].z, kc.c[k].w), m0[k]));
            }
        } else {
            const int qa = r_q[ra], qb = r_q[rbt];
            const bool co_ab = live && __ldg(sc.coinc + qa + colb);
            for (int j = 0; j < trip; ++j) {
                float m0[NMP];
                load_msgs<NMP>(mrow + (size_t)j * NMP, m0);
                const bool cbc = __ldg(sc.coinc + qb + j);
                const bool cac = __ldg(sc.coinc + qa + sg.aoff + j);
#pragma unroll
                for (int k = 0; k < NM; ++k)
                    R[k] = fminf(R[k], cand_value(m0[k], brow[j], th_ab, arow[j], cbc || co_ab, cbc || cac,
                                                  kc.c[k].z, kc.c[k].w, p.l23));
            }
        }
        if (live) {
            const int64_t out = (int64_t)(r_q[ra] + colb - d.pbase) * NM;
#pragma unroll
            for (int k = 0; k < NM; ++k) {
                const float real = __fadd_rn(R[k], state_const(p.l2, kc.c[k].y, sg.g));
                const float eps = __fadd_rn(p.l1W, b_ean[(b - B0) * NM + k]);
                cur[out + k] = fminf(real, eps);
            }
        }
    }
}

// ------------------------------------------------------------------ launchers
size_t dp_batch_smem(const TileGeom &tg, int T, int NM) { return SmemPlan(tg, T, NM).total; }

template <int NM>
static hgm_status launch_nm(const SceneView &v, const InstDesc *dinst, int ninst, float *hist, int64_t L, int layer,
                            bool has_next, bool has_prev, const StepConstB &kc, const float *msg, const DPParams &p,
                            const TileGeom &tg, cudaStream_t s) {
    const size_t smem = dp_batch_smem(tg, p.T, NM);
    static size_t configured[2] = {48 * 1024, 48 * 1024};
    auto kern = has_next ? k_dp_batch<NM, true> : k_dp_batch<NM, false>;
    size_t &cfg = configured[has_next ? 1 : 0];
    if (smem > cfg) {
        HGM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        cfg = smem;
    }
    const dim3 grid((unsigned)tg.ntile, (unsigned)ninst);
    kern<<<grid, KDP_THREADS, smem, s>>>(v, dinst, hist, L, layer, has_prev ? 1 : 0, kc, msg, p, tg);
    return HGM_OK;
}

hgm_status launch_dp_batch(int NM, const SceneView &v, const InstDesc *dinst, int ninst, float *hist, int64_t L,
                           int layer, bool has_next, bool has_prev, const StepConstB &kc, const float *msg,
                           const DPParams &p, const TileGeom &tg, cudaStream_t s) {
#define HGM_NM_CASE(n) case n: return launch_nm<n>(v, dinst, ninst, hist, L, layer, has_next, has_prev, kc, msg, p, tg, s)
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
}

}  // namespace hgm
