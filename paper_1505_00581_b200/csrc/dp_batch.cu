// dp_batch.cu -- K-DP: one recursion step i of PAPER.md Eq. 10 for a batch of
// NM models of equal chain length M against a chunk of windows.
//
// Work item = (window, tile of consecutive b-frames).  Tiles are a host-side
// partition of the scene's frames sized to a shared-memory budget (dense frames
// give short tiles), clipped to each window.  The kernel is PERSISTENT: a few CTAs
// per SM pull items from a counter, and while one item runs its candidate loop the
// inputs of the next item stream in by TMA bulk copies (cp.async.bulk, completion
// on an mbarrier) -- every input of an item is a contiguous range of the scene
// index, the unary table or the alpha layer i+1.
//
// For the states of layer i whose second label b lies in the item's frames:
//   real      alpha_i(b, a)   = min( min_{c in L(b,a)} [ m(b,c) + lambda2 lambda3 Dg(c,b,a) ]
//                                    + lambda2 |g_{i-1} - (t'(b) - t'(a))|,
//                                    lambda1 W^d + alpha_{i+1}(eps, b) )
//   (b, eps)  alpha_i(b, eps) = min( min_c n(b,c), lambda1 W^d + alpha_{i+1}(eps, b) )
//   (eps, b)  alpha_i(eps, b) = min( min_{c in frames (t'(b), t'(b)+T)} w(c), lambda1 W^d + alpha_{i+1}(eps, eps) )
//   (eps,eps) alpha_i(eps,eps)= min( min_{c in window} w(c), lambda1 W^d + alpha_{i+1}(eps, eps) )
//             (each item min-reduces its own frames into the slot with an atomic)
// with L(b,a) = [minnode(t'(b)+1), minnode(t'(a)+T)) (R1-R3),
//   n(b,c) = alpha_{i+1}(c, b) + lambda1 U_i(c)        (Eq. 10 without D)
//   m(b,c) = n(b,c) + lambda2 |g_i - (t'(c) - t'(b))|  (the Delta term of the (i, i-1) edge)
//   w(c)   = alpha_{i+1}(c, eps) + lambda1 U_i(c)
// and D = 0 whenever a label of the triple is the dummy (reading R5).
//
// Per item: wait for the bulk copies; P1 row bookkeeping, segment table (a
// (b-frame, a-frame) segment shares its candidate range), per-frame minima of w;
// P2 segment prefix, message build (one warp per b row: the alpha_{i+1} row,
// lambda1 U and the Delta table give the NM messages of every candidate entry,
// stored with theta(b -> c) as float4s; the (b, eps) minimum is a full-warp
// redux), the dummy-form states; then the next item's copies are issued; P3 the
// state -> segment map; P4 the real states, one per lane, ordered by frame gap so
// the lanes of a warp see near-equal trip counts.  Per candidate: 2 LDS.128
// (messages + theta_bc), 1 LDS (theta_ac), the two scene-angle folds shared by the
// NM models, then per PAIR of models FADD2, FADD2, FMUL2, FFMA2, 2 MUFU.SQRT, FFMA2
// (packed f32x2, sm_100) and a 3-input min over candidate pairs.  States touching a
// coincident pair (R10) take the exact flag-aware loop.
//
// The arithmetic is hgm_device.cuh's (packed ops round like the scalar ones), so the
// backtrack's re-evaluation (backtrack.cu) stays bit-identical.
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
constexpr int NROWI = 6;  // derived row bookkeeping ints per row

__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~(size_t)15; }

struct SmemPlan {
    size_t en, araw, th0, th1, uc, we, tc, ni, rfc, rlc, eb, ee, ftab, rows, bean, fw, dl, seg, map, item, total;
    __host__ __device__ SmemPlan(const TileCaps &c, int T, int NM) {
        size_t o = 0;
        auto take = [&](size_t bytes) {
            const size_t r = o;
            o = align16(o + bytes);
            return r;
        };
        en = take(sizeof(float) * (size_t)entry_floats(NM) * c.NE);
        araw = take(sizeof(float) * ((size_t)NM * c.NE + 8));
        th0 = take(sizeof(float) * ((size_t)c.TH + 8));
        th1 = take(sizeof(float) * ((size_t)c.TH + 8));
        uc = take(sizeof(float) * ((size_t)NM * c.NC + 8));
        we = take(sizeof(float) * ((size_t)NM * c.NC + 8));
        tc = take(sizeof(int) * ((size_t)c.NC + 8));
        ni = take(sizeof(int4) * ((size_t)c.NA + 1));
        rfc = take(sizeof(int) * ((size_t)c.NA + 8));
        rlc = take(sizeof(int) * ((size_t)c.NA + 8));
        eb = take(sizeof(float) * ((size_t)NM * c.NB + 8));
        ee = take(sizeof(float) * ((size_t)NM + 8));
        ftab = take(sizeof(int) * ((size_t)c.FT + 2 * T + 16));
        rows = take(sizeof(int) * NROWI * (size_t)c.NA);
        bean = take(sizeof(float) * (size_t)NM * c.NB);
        fw = take(sizeof(float) * (size_t)NM * (c.FT + T));
        dl = take(sizeof(float) * (size_t)NM * T);
        seg = take(sizeof(Seg) * (size_t)c.FT * (T - 1));
        map = take((size_t)c.NST);
        item = take(2 * sizeof(WorkItem) + 2 * sizeof(InstDesc) + 5 * 8 + 16);  // descriptors, mbarriers, scalars
        total = o;
    }
};

// ------------------------------------------------------------------ TMA bulk copies
__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity) {
    unsigned ok = 0;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    } while (!ok);
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// Up to 12 bulk copies of one item, collected first so the mbarrier is armed with
// the total byte count before any copy is issued.
struct CopyList {
    int n = 0;
    unsigned total = 0;
    void *dst[12];
    const void *src[12];
    unsigned bytes[12];
    __device__ __forceinline__ void add(void *d, const void *s, unsigned b) {
        if (b == 0) return;
        dst[n] = d;
        src[n] = s;
        bytes[n] = b;
        total += b;
        ++n;
    }
    // Elements [g0, g1) of a 4-byte-element array, widened to whole 16-byte units
    // (the allocations carry >= 16 bytes of slack): dst[q] = src[a0 + q], a0 = g0 & ~3.
    // Returns g0 - a0, the index of element g0 in dst.
    template <class T>
    __device__ __forceinline__ int range(void *d, const T *s, int64_t g0, int64_t g1) {
        static_assert(sizeof(T) == 4, "4-byte elements");
        const int64_t a0 = g0 & ~(int64_t)3, a1 = (g1 + 3) & ~(int64_t)3;
        if (g1 > g0) add(d, s + a0, (unsigned)((a1 - a0) * 4));
        return (int)(g0 - a0);
    }
    __device__ __forceinline__ void issue(uint64_t *bar) {
        mbar_expect_tx(bar, total);
        for (int q = 0; q < n; ++q) bulk_g2s(dst[q], src[q], bytes[q], bar);
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

template <int EPF>
__device__ __forceinline__ void ld_entry(const float *__restrict__ src, float (&e)[EPF]) {
#pragma unroll
    for (int q = 0; q < EPF / 4; ++q) {
        const float4 v = reinterpret_cast<const float4 *>(src)[q];
        e[4 * q] = v.x;
        e[4 * q + 1] = v.y;
        e[4 * q + 2] = v.z;
        e[4 * q + 3] = v.w;
    }
}

template <int NM>
__device__ __forceinline__ void st_alpha(float *__restrict__ dst, const float (&v)[NM]) {
    if constexpr (NM % 2 == 0) {
#pragma unroll
        for (int q = 0; q < NM / 2; ++q) reinterpret_cast<float2 *>(dst)[q] = make_float2(v[2 * q], v[2 * q + 1]);
    } else {
#pragma unroll
        for (int q = 0; q < NM; ++q) dst[q] = v[q];
    }
}

// v_k = l23 * sqrt((fb - A1_k)^2 + (fc - K2_k)^2) + m_k for every model k; exactly the
// rounding sequence of cand_value() in hgm_device.cuh, two models per packed op.
template <int NM>
__device__ __forceinline__ void cand_values(float fb, float fc, const float *m, const StepConstB &pc, float l23,
                                            float (&v)[NM]) {
#pragma unroll
    for (int q = 0; q < NM / 2; ++q) {
        const float2 e1 = __fadd2_rn(make_float2(fb, fb), pc.nA1[q]);
        const float2 e2 = __fadd2_rn(make_float2(fc, fc), pc.nK2[q]);
        const float2 qq = __ffma2_rn(e1, e1, __fmul2_rn(e2, e2));
        const float2 s = make_float2(sqrt_approx(qq.x), sqrt_approx(qq.y));
        const float2 r = __ffma2_rn(make_float2(l23, l23), s, make_float2(m[2 * q], m[2 * q + 1]));
        v[2 * q] = r.x;
        v[2 * q + 1] = r.y;
    }
    if constexpr (NM % 2 == 1) {
        constexpr int k = NM - 1;
        const float e1 = __fadd_rn(fb, pc.nA1[k / 2].x);
        const float e2 = __fadd_rn(fc, pc.nK2[k / 2].x);
        v[k] = __fmaf_rn(l23, sqrt_approx(__fmaf_rn(e1, e1, __fmul_rn(e2, e2))), m[k]);
    }
}

// The bulk copies of one item's inputs (producer lane): every range is computed
// first, the item's descriptors are published to shared memory, then the stage's
// mbarrier is armed with the byte total and the copies are issued.
template <int NM, bool kHasNext>
__device__ __forceinline__ void plan_item(const SceneView &sc, WorkItem &w, const InstDesc &d, const float *hist,
                                          int64_t L, int layer, const float *__restrict__ U, int64_t ui_off, int T,
                                          const SmemPlan &sp, unsigned char *smem, int thstage, CopyList &cl) {
    // sources are addressed from the (16-byte aligned) allocation bases
    const int64_t nxo = (int64_t)(layer + 1) * L + d.off;  // alpha layer i+1 of this window in hist
    const int Sw = d.we - d.wb;
    // direction rows x in [A0, B1) of the padded band
    w.th0 = w.qa - cl.range(smem + (thstage ? sp.th1 : sp.th0), sc.theta_pad, w.qa, w.qb1);  // TH[q] = theta_pad[th0 + q]
    if (kHasNext) {  // alpha_{i+1}: rows of the tile's b nodes (padded layout) and the dummy-form slots
        w.araw0 = cl.range(smem + sp.araw, hist, nxo + (int64_t)(w.qb0 - d.ppad) * NM, nxo + (int64_t)(w.qb1 - d.ppad) * NM);
        w.we0 = cl.range(smem + sp.we, hist, nxo + (int64_t)(d.ntail + w.B0 - d.wb) * NM,
                         nxo + (int64_t)(d.ntail + w.Cend - d.wb) * NM);
        w.eb0 = cl.range(smem + sp.eb, hist, nxo + (int64_t)(d.ntail + Sw + w.B0 - d.wb) * NM,
                         nxo + (int64_t)(d.ntail + Sw + w.B1 - d.wb) * NM);
        w.ee0 = cl.range(smem + sp.ee, hist, nxo + (int64_t)(d.ntail + 2 * Sw) * NM,
                         nxo + (int64_t)(d.ntail + 2 * Sw + 1) * NM);
    }
    w.uc0 = cl.range(smem + sp.uc, U, ui_off + (int64_t)w.B0 * NM, ui_off + (int64_t)w.Cend * NM);
    w.tc0 = cl.range(smem + sp.tc, sc.t, w.B0, w.Cend);
    if (w.B1 > w.A0) cl.add(smem + sp.ni, sc.ninfo + w.A0, (unsigned)(sizeof(int4) * (w.B1 - w.A0)));
    w.rf0 = cl.range(smem + sp.rfc, sc.rfc, w.A0, w.B1);
    cl.range(smem + sp.rlc, sc.rlc, w.A0, w.B1);
    // first_tab over frames [F0 - T, F1 + T], clamped to the table
    const int f_lo = max(0, w.F0 - T), f_hi = min(sc.fmax + 1, w.F1 + T);
    w.ft0 = cl.range(smem + sp.ftab, sc.ft, f_lo, f_hi + 1);
    w.flo = f_lo;
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// consumer-only barrier (the producer warp never joins it)
__device__ __forceinline__ void consumers_sync() { asm volatile("bar.sync 1, %0;" ::"n"(KDP_THREADS) : "memory"); }

template <int NM, bool kHasNext>
__global__ void __launch_bounds__(KDP_THREADS + 32, 2) k_dp_fused(SceneView sc, const InstDesc *__restrict__ inst,
                                                             const WorkItem *__restrict__ items, int nitems,
                                                             int *__restrict__ counter, float *__restrict__ hist,
                                                             int64_t L, int layer, int has_prev, StepConstB kc,
                                                             const float *__restrict__ U, int64_t ui_off, DPParams p,
                                                             TileCaps caps) {
    constexpr int EPF = entry_floats(NM);
    extern __shared__ __align__(128) unsigned char smem[];
    const SmemPlan sp(caps, p.T, NM);
    float *EN = reinterpret_cast<float *>(smem + sp.en);
    const float *ARAW = reinterpret_cast<const float *>(smem + sp.araw);
    const float *UC = reinterpret_cast<const float *>(smem + sp.uc);
    const float *WE = reinterpret_cast<const float *>(smem + sp.we);
    const int *TC = reinterpret_cast<const int *>(smem + sp.tc);
    const int4 *NI = reinterpret_cast<const int4 *>(smem + sp.ni);
    const int *RFC = reinterpret_cast<const int *>(smem + sp.rfc);
    const int *RLC = reinterpret_cast<const int *>(smem + sp.rlc);
    const float *EB = reinterpret_cast<const float *>(smem + sp.eb);
    const float *EE = reinterpret_cast<const float *>(smem + sp.ee);
    const int *FTAB = reinterpret_cast<const int *>(smem + sp.ftab);
    int *r_ofs = reinterpret_cast<int *>(smem + sp.rows);  // [NA] offset of row x in TH
    int *r_en = r_ofs + caps.NA;                             // entry index of row x's column 0 in EN
    int *r_q = r_en + caps.NA;                               // qstart[x] (compact band: coincidence flags)
    int *r_qp = r_q + caps.NA;                               // qpad[x] (padded band: alpha slots)
    int *r_fc = r_qp + caps.NA;                              // first / last coincident column
    int *r_lc = r_fc + caps.NA;
    float *b_ean = reinterpret_cast<float *>(smem + sp.bean);  // [NB][NM] lambda1 W^d + alpha_{i+1}(eps, b)
    float *fw = reinterpret_cast<float *>(smem + sp.fw);       // [FT + T][NM] frame minima of w
    float *DL = reinterpret_cast<float *>(smem + sp.dl);       // [T][NM] lambda2 |g_i - dt|
    Seg *seg = reinterpret_cast<Seg *>(smem + sp.seg);
    uint8_t *smap = smem + sp.map;
    WorkItem *s_item = reinterpret_cast<WorkItem *>(smem + sp.item);            // [2] per stage
    InstDesc *s_inst = reinterpret_cast<InstDesc *>(smem + sp.item + 2 * sizeof(WorkItem));  // [2]
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + sp.item + 2 * sizeof(WorkItem) + 2 * sizeof(InstDesc));
    uint64_t *full = bars;         // [2] item inputs landed (producer arrive + TMA bytes)
    uint64_t *empty_in = bars + 2; // single-buffered inputs consumed (after P2)
    uint64_t *empty_th = bars + 3; // [2] direction rows of a stage consumed (after the loop)
    int *s_nst = reinterpret_cast<int *>(bars + 5);
    int *s_claim = s_nst + 1;

    const int T = p.T;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    for (int q = tid; q < T * NM; q += blockDim.x) {
        const int dt = q / NM, k = q - dt * NM;
        DL[q] = delta_term(p.l2, kc.c[k].x, dt);
    }
    if (tid == 0) {
        mbar_init(full, 1);
        mbar_init(full + 1, 1);
        mbar_init(empty_in, 1);
        mbar_init(empty_th, 1);
        mbar_init(empty_th + 1, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp == KDP_WARPS) {  // ---------------- producer warp: claims items, streams their inputs
        if (lane != 0) return;
        for (int n = 0;; ++n) {
            const int s = n & 1;
            int idx;
            WorkItem w{};
            do {  // skip empty slots
                idx = atomicAdd(counter, 1);
                if (idx >= nitems) break;
                w = items[idx];
            } while (w.F1 <= w.F0);
            InstDesc d{};
            CopyList cl;
            if (idx < nitems) {
                d = inst[w.inst];
                plan_item<NM, kHasNext>(sc, w, d, hist, L, layer, U, ui_off, T, sp, smem, s, cl);
            } else {
                w.inst = -1;
            }
            if (n >= 1) mbar_wait(empty_in, (n - 1) & 1);       // item n-1 finished P2
            if (n >= 2) mbar_wait(empty_th + s, ((n - 2) >> 1) & 1);  // item n-2 finished its loop
            s_item[s] = w;
            s_inst[s] = d;
            if (w.inst < 0) {
                mbar_arrive(full + s);
                return;
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // earlier generic accesses before async writes
            cl.issue(full + s);
        }
    }

    // ---------------- consumer warps
    for (int n = 0;; ++n) {
        const int stage = n & 1;
        mbar_wait(full + stage, (n >> 1) & 1);
        const WorkItem w = s_item[stage];
        if (w.inst < 0) break;
        const InstDesc d = s_inst[stage];
        const float *TH = reinterpret_cast<const float *>(smem + (stage ? sp.th1 : sp.th0));
        const int F0 = w.F0, F1 = w.F1, B0 = w.B0, B1 = w.B1, A0 = w.A0;
        const int NR = B1 - A0, NBr = B1 - B0;
        const int Sw = d.we - d.wb;
        const int wend = d.o + caps.W;
        float *cur = hist + (int64_t)layer * L + d.off;
        const int nseg = (F1 - F0) * (T - 1);
        auto first = [&](int f) { return f <= 0 ? 0 : (f > sc.fmax ? sc.S : FTAB[w.ft0 + (f - w.flo)]); };

        // ---------------- P1: segment table + prefix (warp 0); row bookkeeping, frame minima of w (warps 1..)
        if (warp == 0) {  // segments, gap-major: long candidate ranges first
            int carry = 0;
            for (int r0 = 0; r0 < nseg; r0 += 32) {
                const int r = r0 + lane;
                Seg sg{};
                int cnt = 0;
                if (r < nseg) {
                    const int g = 1 + r / (F1 - F0);
                    const int f = F0 + r % (F1 - F0);
                    if (f - g >= d.o) {
                        sg.g = g;
                        sg.b0 = first(f);
                        sg.nb = first(f + 1) - sg.b0;
                        sg.a0 = first(f - g);
                        sg.f1a = first(f - g + 1);
                        const int c0 = first(f + 1);
                        sg.trip = max(0, min(first(f - g + T), d.we) - c0);
                        sg.aoff = c0 - sg.f1a;
                        sg.inv = sg.nb > 1 ? (unsigned)((0x100000000ull + sg.nb - 1) / sg.nb) : 0u;
                        cnt = sg.nb * (sg.f1a - sg.a0);
                    }
                }
                const int incl = warp_incl_scan(cnt, lane);
                sg.start = carry + incl - cnt;
                if (r < nseg) seg[r] = sg;
                carry += __shfl_sync(0xffffffffu, incl, 31);
            }
            if (lane == 0) {
                *s_nst = carry;
                *s_claim = 0;
            }
        } else {
            const int t1 = tid - 32;
            for (int r = t1; r < NR; r += KDP_THREADS - 32) {
                const int4 ni = NI[r];  // (t', minnode(t'+1), qstart, qpad)
                r_ofs[r] = ni.w - w.th0;  // TH[q] holds theta_pad[th0 + q]
                r_en[r] = ni.w - w.qb0;
                r_q[r] = ni.z;
                r_qp[r] = ni.w;
                r_fc[r] = RFC[w.rf0 + r];  // whole (unclipped) row: conservative
                r_lc[r] = RLC[w.rf0 + r];
            }
            const int nfw = min(F1 + T - 1, wend) - F0;  // frames [F0, F1 + T - 1) inside the window
            for (int q = t1; q < nfw * NM; q += KDP_THREADS - 32) {
                const int fi = q / NM, k = q - fi * NM, f = F0 + fi;
                float wm = INFINITY;
                const int c1 = first(f + 1);
                for (int c = first(f); c < c1; ++c)
                    wm = fminf(wm, msg_n(kHasNext ? WE[w.we0 + (c - B0) * NM + k] : 0.f, p.l1,
                                         UC[w.uc0 + (c - B0) * NM + k]));
                fw[q] = wm;
            }
        }
        consumers_sync();

        // ---------------- P2: state -> segment map, messages + (b, eps), (eps, b), (eps, eps)
        const int nst = *s_nst;
        for (int s = warp; s < nseg; s += KDP_WARPS) {
            const int st0 = seg[s].start, cnt = (s + 1 < nseg ? seg[s + 1].start : nst) - st0;
            for (int q = lane; q < cnt; q += 32) smap[st0 + q] = (uint8_t)s;
        }
        for (int rb = warp; rb < NBr; rb += KDP_WARPS) {  // one warp per b row
            const int r = rb + (B0 - A0);
            const int tb = NI[r].x, c0 = NI[r].y;
            const int len = min(first(tb + T), d.we) - c0;  // candidates of row b in this window (R1, R2)
            const int e0 = r_en[r], t0 = r_ofs[r];
            float mn[NM];
#pragma unroll
            for (int k = 0; k < NM; ++k) mn[k] = INFINITY;
            for (int j = lane; j < len; j += 32) {
                const int e = e0 + j, cc = c0 + j - B0;
                const int dt = TC[w.tc0 + cc] - tb;
                float ent[EPF];
#pragma unroll
                for (int k = 0; k < NM; ++k) {
                    const float n = msg_n(kHasNext ? ARAW[w.araw0 + e * NM + k] : 0.f, p.l1, UC[w.uc0 + cc * NM + k]);
                    mn[k] = fminf(mn[k], n);
                    ent[k] = __fadd_rn(n, DL[dt * NM + k]);  // msg_m
                }
                ent[NM] = TH[t0 + j];
#pragma unroll
                for (int k = NM + 1; k < EPF; ++k) ent[k] = 0.f;
#pragma unroll
                for (int q = 0; q < EPF / 4; ++q)
                    reinterpret_cast<float4 *>(EN + (size_t)e * EPF)[q] =
                        make_float4(ent[4 * q], ent[4 * q + 1], ent[4 * q + 2], ent[4 * q + 3]);
            }
            float ean = 0.f, bm = INFINITY;
#pragma unroll
            for (int k = 0; k < NM; ++k) {  // n >= 0: float order = unsigned bit order
                const float v = __uint_as_float(__reduce_min_sync(0xffffffffu, __float_as_uint(mn[k])));
                if (lane == k) bm = v;
            }
            if (lane < NM) {
                ean = __fadd_rn(p.l1W, kHasNext ? EB[w.eb0 + rb * NM + lane] : 0.f);  // lambda1 W^d + alpha_{i+1}(eps, b)
                b_ean[rb * NM + lane] = ean;
                cur[(int64_t)(d.ntail + B0 + rb - d.wb) * NM + lane] = fminf(bm, ean);  // (b, eps)
            }
        }
        for (int q = tid; q < NBr * NM; q += KDP_THREADS) {  // (eps, b): frames (t'(b), t'(b) + T) inside the window
            const int rb = q / NM, k = q - rb * NM;
            const int tb = NI[rb + (B0 - A0)].x;
            float r = INFINITY;
            const int f1 = min(tb + T, wend);
            for (int f = tb + 1; f < f1; ++f) r = fminf(r, fw[(f - F0) * NM + k]);
            cur[(int64_t)(d.ntail + Sw + B0 + rb - d.wb) * NM + k] =
                fminf(r, __fadd_rn(p.l1W, kHasNext ? EE[w.ee0 + k] : 0.f));
        }
        if (tid < NM) {  // (eps, eps): this item's frames, min-reduced into the slot (reset to +inf by step i+1)
            float r = __fadd_rn(p.l1W, kHasNext ? EE[w.ee0 + tid] : 0.f);
            for (int f = F0; f < F1; ++f) r = fminf(r, fw[(f - F0) * NM + tid]);
            atomicMin(reinterpret_cast<unsigned *>(cur + (int64_t)(d.ntail + 2 * Sw) * NM + tid), __float_as_uint(r));
            if (has_prev && F0 == d.o)  // the next step's slot starts at +inf
                (cur - L)[(int64_t)(d.ntail + 2 * Sw) * NM + tid] = INFINITY;
        }
        consumers_sync();
        if (tid == 0) mbar_arrive(empty_in);  // the producer may refill the single-buffered inputs

        // ---------------- P4: real states (b, a)
        for (;;) {  // warps claim 32-state groups (gap-major order: longest trips first)
            int s0 = 0;
            if (lane == 0) s0 = atomicAdd(s_claim, 32);
            s0 = __shfl_sync(0xffffffffu, s0, 0);
            if (s0 >= nst) break;
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
            const float *erow = EN + (size_t)r_en[rbt] * EPF;
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
                    float e0[EPF], e1[EPF];
                    ld_entry<EPF>(erow + (size_t)j * EPF, e0);
                    ld_entry<EPF>(erow + (size_t)(j + 1) * EPF, e1);
                    const float ac0 = arow[j], ac1 = arow[j + 1];
                    float v0[NM], v1[NM];
                    cand_values<NM>(fold(e0[NM], th_ab), fold(e0[NM], ac0), e0, kc, p.l23, v0);
                    cand_values<NM>(fold(e1[NM], th_ab), fold(e1[NM], ac1), e1, kc, p.l23, v1);
#pragma unroll
                    for (int k = 0; k < NM; ++k) R[k] = min3(R[k], v0[k], v1[k]);
                }
                if (j < trip) {
                    float e0[EPF];
                    ld_entry<EPF>(erow + (size_t)j * EPF, e0);
                    float v0[NM];
                    cand_values<NM>(fold(e0[NM], th_ab), fold(e0[NM], arow[j]), e0, kc, p.l23, v0);
#pragma unroll
                    for (int k = 0; k < NM; ++k) R[k] = fminf(R[k], v0[k]);
                }
            } else {
                const int qa = r_q[ra], qb = r_q[rbt];
                const bool co_ab = live && __ldg(sc.coinc + qa + colb);
                for (int j = 0; j < trip; ++j) {
                    float e0[EPF];
                    ld_entry<EPF>(erow + (size_t)j * EPF, e0);
                    const bool cbc = __ldg(sc.coinc + qb + j);
                    const bool cac = __ldg(sc.coinc + qa + sg.aoff + j);
#pragma unroll
                    for (int k = 0; k < NM; ++k)
                        R[k] = fminf(R[k], cand_value(e0[k], e0[NM], th_ab, arow[j], cbc || co_ab, cbc || cac,
                                                      kc.c[k].z, kc.c[k].w, p.l23));
                }
            }
            if (live) {
                float out[NM];
#pragma unroll
                for (int k = 0; k < NM; ++k) {
                    const float real = __fadd_rn(R[k], state_const(p.l2, kc.c[k].y, sg.g));
                    out[k] = fminf(real, b_ean[(b - B0) * NM + k]);
                }
                st_alpha<NM>(cur + (int64_t)(r_qp[ra] + colb - d.ppad) * NM, out);
            }
        }
        consumers_sync();
        if (tid == 0) mbar_arrive(empty_th + stage);  // this stage's direction rows may be refilled
    }
}

// (eps, eps) slots of the first layer of a chunk start at +inf (later layers: reset by K-DP)
__global__ void k_init_ee(const InstDesc *__restrict__ inst, int ninst, float *__restrict__ hist, int64_t L,
                          int layer, int NM) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= ninst * NM) return;
    const int k = q / NM, m = q - k * NM;
    const InstDesc d = inst[k];
    hist[(int64_t)layer * L + d.off + (int64_t)(d.ntail + 2 * (d.we - d.wb)) * NM + m] = INFINITY;
}

// Work items of a chunk: slot x of window k is the x-th global tile meeting the
// window's frames, clipped to them; descriptors are valid for every step.
__global__ void k_items(SceneView sc, const InstDesc *__restrict__ inst, int ninst, int W, int T,
                        const int32_t *__restrict__ gstart, const int32_t *__restrict__ tile_of, int tf_lo,
                        int slots, WorkItem *items) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= ninst * slots) return;
    const int k = q / slots, x = q - k * slots;
    const InstDesc d = inst[k];
    const int gt = __ldg(tile_of + (d.o - tf_lo)) + x;
    WorkItem w{};
    w.inst = k;
    w.F0 = max(__ldg(gstart + gt), d.o);
    w.F1 = min(__ldg(gstart + gt + 1), d.o + W);
    if (w.F0 >= d.o + W) {  // no such tile: empty item (F1 <= F0)
        w.F0 = w.F1 = d.o + W;
    }
    w.B0 = sc.first(w.F0);
    w.B1 = sc.first(w.F1);
    w.A0 = max(sc.first(w.F0 - T + 1), d.wb);
    w.Cend = min(sc.first(w.F1 + T - 1), d.we);
    w.qa = __ldg(sc.qpad + w.A0);
    w.qb0 = __ldg(sc.qpad + w.B0);
    w.qb1 = __ldg(sc.qpad + w.B1);
    items[q] = w;
}

// ------------------------------------------------------------------ launchers
size_t dp_batch_smem(const TileCaps &c, int T, int NM) { return SmemPlan(c, T, NM).total; }

template <int NM>
static hgm_status launch_nm(const SceneView &v, const InstDesc *dinst, const WorkItem *items, int nitems,
                            int *counter, float *hist, int64_t L, int layer, bool has_next, bool has_prev,
                            const StepConstB &kc, const float *U, int64_t ui_off, const DPParams &p,
                            const TileCaps &caps, cudaStream_t s) {
    const size_t smem = dp_batch_smem(caps, p.T, NM);
    auto kern = has_next ? k_dp_fused<NM, true> : k_dp_fused<NM, false>;
    static int configured[2] = {0, 0};
    static int blocks_per_sm[2] = {0, 0};
    const int h = has_next ? 1 : 0;
    if ((int)smem > configured[h]) {
        HGM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        configured[h] = (int)smem;
        HGM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm[h], kern, KDP_THREADS + 32, smem));
    }
    int dev = 0, nsm = 0;
    HGM_CUDA(cudaGetDevice(&dev));
    HGM_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    const int grid = std::max(1, std::min(nitems, std::max(1, blocks_per_sm[h]) * nsm));
    kern<<<grid, KDP_THREADS + 32, smem, s>>>(v, dinst, items, nitems, counter, hist, L, layer, has_prev ? 1 : 0, kc, U,
                                         ui_off, p, caps);
    return HGM_OK;
}

hgm_status launch_dp_batch(int NM, const SceneView &v, const InstDesc *dinst, const WorkItem *items, int nitems,
                           int *counter, float *hist, int64_t L, int layer, bool has_next, bool has_prev,
                           const StepConstB &kc, const float *U, int64_t ui_off, const DPParams &p,
                           const TileCaps &caps, cudaStream_t s) {
#define HGM_NM_CASE(n)                                                                                             \
    case n:                                                                                                        \
        return launch_nm<n>(v, dinst, items, nitems, counter, hist, L, layer, has_next, has_prev, kc, U, ui_off, p, \
                            caps, s)
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

hgm_status launch_items(const SceneView &v, const InstDesc *dinst, int ninst, int W, int T, const int32_t *gstart,
                        const int32_t *tile_of, int tf_lo, int slots, WorkItem *items, cudaStream_t s) {
    const int n = ninst * slots;
    if (n > 0) k_items<<<(n + 255) / 256, 256, 0, s>>>(v, dinst, ninst, W, T, gstart, tile_of, tf_lo, slots, items);
    return HGM_OK;
}

hgm_status launch_init_ee(const InstDesc *dinst, int ninst, float *hist, int64_t L, int layer, int NM,
                          cudaStream_t s) {
    const int n = ninst * NM;
    if (n > 0) k_init_ee<<<(n + 255) / 256, 256, 0, s>>>(dinst, ninst, hist, L, layer, NM);
    return HGM_OK;
}

}  // namespace hgm
