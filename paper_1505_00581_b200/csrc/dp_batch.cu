// dp_batch.cu -- K-DP: one recursion step (Eq. 10) for a batch of NM
// models of equal chain length M against one window, one CTA per (window, tile
// of FT consecutive b-frames), one launch per step i.
//
//   alpha^k_i(b, a) = min( min_{c in L(b,a)} [ m^k(b,c) + lambda2 lambda3 Dg^k(c,b,a) ]
//                          + lambda2 |g^k_{i-1} - (t'(b) - t'(a))|,
//                          lambda1 W^d + alpha^k_{i+1}(eps, b) )
// with L(b,a) = [minnode(t'(b)+1), minnode(t'(a)+T)) (R1-R3),
// the hoisted message m^k(b,c) = n^k(b,c) + lambda2 |g^k_i - (t'(c) - t'(b))| and
// n^k(b,c) = alpha^k_{i+1}(c, b) + lambda1 U^k_i(c) (hgm_device.cuh).
//
// The partial messages n of step i are written by the EPILOGUE of step i+1: the
// thread that produces alpha_{i+1}(c, b) also emits n_i(b, c) into a
// double-buffered message buffer (padded band order), so the alpha layer is
// never re-read to build messages.  This kernel then
//   phase 0  stages its operand rows with two cp.async range copies (direction
//            rows x in [A0, B1) from the padded band, message rows b in [B0, B1))
//            plus row bookkeeping, the node frames and the per-node term
//            w(c) = alpha_{i+1}(c, eps) + lambda1 U_i(c) of its candidate range;
//   phase 1  segment table of the real states (one (b-frame, a-frame) segment
//            shares its candidate range) and per-frame minima of w;
//   phase 2  converts the staged n rows to m in place (the Delta term is a
//            (gap, model) table with the exact arithmetic of msg_m) and reduces
//            the dummy-form states (b, eps), (eps, b) and (eps, eps) of R5;
//   phase 3  evaluates the real states, one per lane, ordered by frame gap, the
//            scene-only work (direction reads, both angle folds) shared by the
//            NM models; the epilogue writes alpha_i (history for K-BT) and the
//            next step's n_{i-1}(a, b) = alpha_i(b, a) + lambda1 U_{i-1}(b).
// States touching a coincident pair (R10) take the exact flag-aware loop.
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
    size_t first, th, mt, rows, brows, cnodes, dtab, fm, seg, map, total;
    __host__ __device__ SmemPlan(const TileGeom &tg, int T, int NM) {
        first = 0;
        th = align16(first + sizeof(int) * (size_t)(tg.FT + 2 * T + 2));
        mt = align16(th + sizeof(float) * (size_t)tg.TH);
        rows = align16(mt + sizeof(float) * (size_t)nm_pad(NM) * tg.MT);
        brows = align16(rows + sizeof(int) * 8 * (size_t)tg.NA);
        cnodes = align16(brows + sizeof(float) * 2 * (size_t)NM * tg.NB);
        dtab = align16(cnodes + sizeof(int) * (1 + (size_t)NM) * tg.NA);
        fm = align16(dtab + sizeof(float) * (size_t)NM * T);
        seg = align16(fm + sizeof(float) * (size_t)NM * (tg.FT + T));
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
// (a 5-CTA/SM register cap was measured: it spills and runs 1.5x slower)
__global__ void __launch_bounds__(KDP_THREADS) k_dp_batch(SceneView sc, const InstDesc *__restrict__ inst,
                                                          float *__restrict__ hist, int64_t L, int layer,
                                                          StepConstB kc, const float *__restrict__ Ui,
                                                          const float *__restrict__ Uprev,
                                                          const float *__restrict__ msg_in,
                                                          float *__restrict__ msg_out, DPParams p, TileGeom tg) {
    constexpr int NMP = nm_pad(NM);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const SmemPlan sp(tg, p.T, NM);
    int *s_first = reinterpret_cast<int *>(smem_raw + sp.first);  // minnode(f), f in [F0-T, F1+T]
    float *TH = reinterpret_cast<float *>(smem_raw + sp.th);
    float *MT = reinterpret_cast<float *>(smem_raw + sp.mt);
    int *r_ofs = reinterpret_cast<int *>(smem_raw + sp.rows);  // [NA] offset of row x in TH
    int *r_q = r_ofs + tg.NA;                                     // qstart[x] (compact band: state index)
    int *r_mo = r_q + tg.NA;                                      // offset of row x in MT / message buffers
    int *r_fc = r_mo + tg.NA;                                     // first / last coincident column
    int *r_lc = r_fc + tg.NA;
    int *r_t = r_lc + tg.NA;   // t'(x)
    int *r_f1 = r_t + tg.NA;   // minnode(t'(x)+1)
    int *r_len = r_f1 + tg.NA; // window-clipped row length
    float *b_ean = reinterpret_cast<float *>(smem_raw + sp.brows);  // [NB][NM] alpha_{i+1}(eps, b)
    float *b_up = b_ean + tg.NB * NM;                               // [NB][NM] U_{i-1}(b)
    int *c_t = reinterpret_cast<int *>(smem_raw + sp.cnodes);       // [NA] t'(c) of the candidate nodes
    float *c_w = reinterpret_cast<float *>(c_t + tg.NA);           // [NA][NM] w(c)
    float *dtab = reinterpret_cast<float *>(smem_raw + sp.dtab);    // [T][NM] lambda2 |g_i - dt|
    float *fmin_ = reinterpret_cast<float *>(smem_raw + sp.fm);     // [FT+T][NM] frame minima of w
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
    const int CR0 = sc.first(F0 + 1), CR1 = min(sc.first(F1 + T - 1), d.we);  // candidate nodes of the b rows
    const int NR = B1 - A0, NBr = B1 - B0, NC = max(0, CR1 - CR0);
    const int Sw = d.we - d.wb;
    float *cur = hist + (int64_t)layer * L + d.off;
    const float *nxt = kHasNext ? hist + (int64_t)(layer + 1) * L + d.off : nullptr;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nseg = tg.FT * (T - 1);
    const int FL = F0 - T;

    // ---------------- phase 0: staging (independent loads)
    int64_t th0 = 0, mt0 = 0;  // source index held by TH[0] / MT[0]
    if (NR > 0) {
        const int qa = __ldg(sc.qpad + A0), qb0 = __ldg(sc.qpad + B0), qb1 = __ldg(sc.qpad + B1);
        th0 = copy_range(TH, sc.theta_pad, qa, qb1, tid);
        if (NBr > 0)
            mt0 = copy_range(MT, msg_in + d.moff, (int64_t)(qb0 - d.ppad) * NMP, (int64_t)(qb1 - d.ppad) * NMP, tid);
        asm volatile("cp.async.commit_group;");
    }
    for (int q = tid; q <= F1 + T - FL; q += KDP_THREADS) s_first[q] = sc.first(FL + q);
    for (int r = tid; r < NR; r += KDP_THREADS) {
        const int x = A0 + r;
        const int qp = __ldg(sc.qpad + x);
        r_ofs[r] = (int)(qp - th0);
        r_mo[r] = (int)((int64_t)(qp - d.ppad) * NMP - mt0);
        r_q[r] = sc.qstart[x];
        r_fc[r] = __ldg(sc.rfc + x);  // whole (unclipped) row: conservative
        r_lc[r] = __ldg(sc.rlc + x);
        r_t[r] = sc.t[x];
        if (x >= B0) {
#pragma unroll
            for (int k = 0; k < NM; ++k) {
                b_ean[(x - B0) * NM + k] = kHasNext ? nxt[(int64_t)(d.np + Sw + (x - d.wb)) * NM + k] : 0.f;
                b_up[(x - B0) * NM + k] = Uprev ? __ldg(Uprev + (int64_t)x * NM + k) : 0.f;
            }
        }
    }
    for (int q = tid; q < NC * NM; q += KDP_THREADS) {
        const int ci = q / NM, k = q - ci * NM, c = CR0 + ci;
        if (k == 0) c_t[ci] = __ldg(sc.t + c);
        c_w[q] = msg_n(kHasNext ? nxt[(int64_t)(d.np + (c - d.wb)) * NM + k] : 0.f, p.l1,
                       __ldg(Ui + (int64_t)c * NM + k));
    }
    for (int dt = tid; dt < T; dt += KDP_THREADS) {
#pragma unroll
        for (int k = 0; k < NM; ++k) dtab[dt * NM + k] = delta_term(p.l2, kc.c[k].x, dt);  // static k: no local copy
    }
    __syncthreads();
    auto FIRST = [&](int f) { return s_first[f - FL]; };

    // ---------------- phase 1: row lengths, segments, frame minima of w
    for (int r = tid; r < NR; r += KDP_THREADS) {
        const int f1 = FIRST(r_t[r] + 1);
        r_f1[r] = f1;
        r_len[r] = max(0, min(FIRST(r_t[r] + T), d.we) - f1);
    }
    for (int s = tid; s < nseg; s += KDP_THREADS) {  // gap-major: long candidate ranges first
        Seg sg{};
        int cnt = 0;
        const int g = 1 + s / tg.FT;
        const int f = F0 + s % tg.FT;
        if (f < F1 && f - g >= d.o) {
            sg.g = g;
            sg.b0 = FIRST(f);
            sg.nb = FIRST(f + 1) - sg.b0;
            sg.a0 = FIRST(f - g);
            sg.f1a = FIRST(f - g + 1);
            const int c0 = FIRST(f + 1);
            sg.trip = max(0, min(FIRST(f - g + T), d.we) - c0);
            sg.aoff = c0 - sg.f1a;
            sg.inv = sg.nb > 1 ? (unsigned)((0x100000000ull + sg.nb - 1) / sg.nb) : 0u;
            cnt = sg.nb * (sg.f1a - sg.a0);
        }
        sg.start = cnt;  // count; prefix below
        seg[s] = sg;
    }
    const int NF = F1 + T - 1 - (F0 + 1);  // frames (F0, F1+T-1)
    for (int q = tid; q < NF * NM; q += KDP_THREADS) {
        const int fi = q / NM, k = q - fi * NM;
        const int f = F0 + 1 + fi;
        const int c1 = min(FIRST(f + 1), d.we);
        float w = INFINITY;
        for (int c = FIRST(f); c < c1; ++c) w = fminf(w, c_w[(c - CR0) * NM + k]);
        fmin_[q] = w;
    }
    asm volatile("cp.async.wait_all;");
    __syncthreads();

    // ---------------- phase 2: segment prefix; n -> m in place; dummy-form states
    if (warp == KDP_WARPS - 1) {
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
    for (int rb = warp; rb < NBr; rb += KDP_WARPS) {
        const int r = B0 - A0 + rb;
        const int b = B0 + rb;
        const int len = r_len[r], f1 = r_f1[r], tb = r_t[r];
        float *row = MT + r_mo[r];
        unsigned nmin[NM];
#pragma unroll
        for (int k = 0; k < NM; ++k) nmin[k] = 0x7f800000u;
        for (int j0 = 0; j0 < len; j0 += 32) {
            const int j = j0 + lane;
            float n[NMP];
#pragma unroll
            for (int k = 0; k < NMP; ++k) n[k] = INFINITY;
            if (j < len) {
                load_msgs<NMP>(row + (size_t)j * NMP, n);
                const float *dt = dtab + (c_t[f1 + j - CR0] - tb) * NM;
                float m[NM];
#pragma unroll
                for (int k = 0; k < NM; ++k) m[k] = __fadd_rn(n[k], dt[k]);  // == msg_m(n, l2, g_i, dt)
                store_msgs<NM>(row + (size_t)j * NMP, m);
            }
#pragma unroll
            for (int k = 0; k < NM; ++k) nmin[k] = min(nmin[k], __reduce_min_sync(0xffffffffu, __float_as_uint(n[k])));
        }
        if (lane < NM) {
            const int k = lane;
            float nb = INFINITY;
#pragma unroll
            for (int q = 0; q < NM; ++q)
                if (q == k) nb = __uint_as_float(nmin[q]);
            cur[(int64_t)(d.np + (b - d.wb)) * NM + k] = fminf(nb, __fadd_rn(p.l1W, b_ean[rb * NM + k]));  // (b, eps)
            float ea = INFINITY;  // (eps, b): candidates in frames (t'(b), t'(b)+T) inside the window
            const int fhi = min(tb + T, wend);
            for (int f = tb + 1; f < fhi; ++f) ea = fminf(ea, fmin_[(f - F0 - 1) * NM + k]);
            const float ee_next = kHasNext ? nxt[(int64_t)(d.np + 2 * Sw) * NM + k] : 0.f;
            cur[(int64_t)(d.np + Sw + (b - d.wb)) * NM + k] = fminf(ea, __fadd_rn(p.l1W, ee_next));
        }
    }
    if (blockIdx.x == 0 && warp == 0) {  // (eps, eps), owned by tile 0
#pragma unroll
        for (int k = 0; k < NM; ++k) {
            float r = INFINITY;
            for (int c = d.wb + lane; c < d.we; c += 32)
                r = fminf(r, msg_n(kHasNext ? nxt[(int64_t)(d.np + (c - d.wb)) * NM + k] : 0.f, p.l1,
                                   __ldg(Ui + (int64_t)c * NM + k)));
            r = warp_min(r);
            if (lane == 0)
                cur[(int64_t)(d.np + 2 * Sw) * NM + k] =
                    fminf(r, __fadd_rn(p.l1W, kHasNext ? nxt[(int64_t)(d.np + 2 * Sw) * NM + k] : 0.f));
        }
    }
    __syncthreads();
    const int nst = s_nst;
    for (int s = warp; s < nseg; s += KDP_WARPS) {  // state index -> segment id
        const Seg &sg = seg[s];
        const int cnt = (s + 1 < nseg ? seg[s + 1].start : nst) - sg.start;
        for (int q = lane; q < cnt; q += 32) smap[sg.start + q] = (uint8_t)s;
    }
    __syncthreads();

    // ---------------- phase 3: real states (b, a)
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
            float al[NM], nn[NM];
#pragma unroll
            for (int k = 0; k < NM; ++k) {
                const float real = __fadd_rn(R[k], state_const(p.l2, kc.c[k].y, sg.g));
                const float eps = __fadd_rn(p.l1W, b_ean[(b - B0) * NM + k]);
                al[k] = fminf(real, eps);
                cur[out + k] = al[k];
                nn[k] = msg_n(al[k], p.l1, b_up[(b - B0) * NM + k]);  // n_{i-1}(a, b)
            }
            if (msg_out) store_msgs<NM>(msg_out + d.moff + (int64_t)r_mo[ra] + mt0 + (int64_t)colb * NMP, nn);
        }
    }
}

// ------------------------------------------------------------------ launchers
size_t dp_batch_smem(const TileGeom &tg, int T, int NM) { return SmemPlan(tg, T, NM).total; }

template <int NM>
static hgm_status launch_nm(const SceneView &v, const InstDesc *dinst, int ninst, float *hist, int64_t L, int layer,
                            bool has_next, const StepConstB &kc, const float *Ui, const float *Uprev,
                            const float *msg_in, float *msg_out, const DPParams &p, const TileGeom &tg,
                            cudaStream_t s) {
    const size_t smem = dp_batch_smem(tg, p.T, NM);
    static size_t configured[2] = {48 * 1024, 48 * 1024};
    auto kern = has_next ? k_dp_batch<NM, true> : k_dp_batch<NM, false>;
    size_t &cfg = configured[has_next ? 1 : 0];
    if (smem > cfg) {
        HGM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        cfg = smem;
    }
    const dim3 grid((unsigned)tg.ntile, (unsigned)ninst);
    kern<<<grid, KDP_THREADS, smem, s>>>(v, dinst, hist, L, layer, kc, Ui, Uprev, msg_in, msg_out, p, tg);
    return HGM_OK;
}

hgm_status launch_dp_batch(int NM, const SceneView &v, const InstDesc *dinst, int ninst, float *hist, int64_t L,
                           int layer, bool has_next, const StepConstB &kc, const float *Ui, const float *Uprev,
                           const float *msg_in, float *msg_out, const DPParams &p, const TileGeom &tg,
                           cudaStream_t s) {
#define HGM_NM_CASE(n) \
    case n: return launch_nm<n>(v, dinst, ninst, hist, L, layer, has_next, kc, Ui, Uprev, msg_in, msg_out, p, tg, s)
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
