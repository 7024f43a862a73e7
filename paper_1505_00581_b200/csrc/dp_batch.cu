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
// state -> segment map; P4 the real states, one per lane, segments in descending
// order of their trip counts so the lanes of a warp see near-equal trips.  Per candidate: 2 LDS.128
// (messages + theta_bc), 1 LDS (theta_ac), the two scene-angle folds shared by the
// NM models, then per PAIR of models FADD2, FADD2, FMUL2, FFMA2, 2 MUFU.SQRT, FFMA2
// (packed f32x2, sm_100) and a 3-input min over candidate pairs.  States touching a
// coincident pair (R10) take the exact flag-aware loop.
//
// The arithmetic is hgm_device.cuh's (packed ops round like the scalar ones), so the
// backtrack's re-evaluation (backtrack.cu) stays bit-identical.
#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "dp_kdp.cuh"

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

constexpr int KDP_THREADS = 256;               // compute warps (12 measured 3 % slower)
constexpr int KDP_WARPS = KDP_THREADS / 32;
constexpr int KDP_BLOCK = KDP_THREADS + 32;      // + one copy warp (claims items, issues their TMA copies)
constexpr int NROWI = 6;  // derived row bookkeeping ints per row


// Per-item bookkeeping that does not change from step to step (computed once per
// chunk by k_item_prep, copied into the stage with the item's other inputs):
//   nst | segments (with prefix starts) | row tables | state -> segment map
struct BookPlan {
    size_t nst, seg, rows, map, total;
    __host__ __device__ BookPlan(const TileCaps &c, int T) {
        size_t o = 0;
        auto take = [&](size_t bytes) {
            const size_t r = o;
            o = align16(o + bytes);
            return r;
        };
        nst = take(16);
        // <= 255 segments per item (the host tiling caps them: uint8 state -> segment map)
        seg = take(sizeof(Seg) * (size_t)std::min(c.FT * (T - 1), 256));
        rows = take(sizeof(int) * NROWI * (size_t)c.NA);
        map = take((size_t)c.NST);
        total = o;
    }
};

// One STAGE holds everything of one work item, laid out for that item's sizes: its
// candidate entries (the alpha_{i+1} rows land there by TMA in the layer's own layout
// and become messages in place), its direction rows, the small raw inputs, its
// bookkeeping record and the dummy terms of its b rows.  Byte offsets within the stage:
struct StageLayout {
    int en, th, tb, uc, we, tc, ni, eb, ee, ftab, bk, bean, total;
    StageLayout() = default;
    // NE entries, NTH direction floats, NC candidate nodes, NA rows, NB b nodes, FT b-frames
    __host__ __device__ StageLayout(int NE, int NTH, int NC, int NA, int NB, int FT, int T, int NM, int book) {
        // NE entries (and theta of the b rows), NTH direction floats of the a rows
        const int EPF = entry_floats(NM);
        int o = 0;
        auto take = [&](long long bytes) {
            const int r = o;
            o = (int)align16((size_t)(o + bytes));
            return r;
        };
        en = take(4LL * EPF * NE);
        th = take(4LL * (NTH + 8));  // + 8: the copies widen ranges to whole 16-byte units
        tb = take(4LL * (NE + 8));
        uc = take(4LL * (NM * NC + 8));
        we = take(4LL * (EPF * NC + 8));
        tc = take(4LL * (NC + 8));
        ni = take(16LL * (NB + 1));  // node info of the b rows
        eb = take(4LL * (EPF * NB + 8));
        ee = take(4LL * (EPF + 8));
        ftab = take(4LL * (FT + 2 * T + 16));
        bk = take(book);
        bean = take(4LL * NM * NB);
        total = o;
    }
};

__host__ __device__ inline StageLayout item_layout(const WorkItem &w, int T, int NM, int book) {
    return StageLayout(w.qb1 - w.qb0, w.qa1 - w.qa, w.Cend - w.B0, w.nA + (w.B1 - w.B0), w.B1 - w.B0, w.F1 - w.F0, T,
                       NM, book);
}

// Shared memory: two stages of caps.STAGE bytes (the largest item layout of the call;
// while one item is processed the copies of the next one land in the other stage),
// the copy warp's frame minima, the Delta table and the control block.
struct SmemPlan {
    size_t stage[3], fw, dl, sc, ctl, total;
    __host__ __device__ SmemPlan(const TileCaps &c, int T, int NM) {
        size_t o = 0;
        auto take = [&](size_t bytes) {
            const size_t r = o;
            o = align16(o + bytes);
            return r;
        };
        stage[0] = take((size_t)c.STAGE);
        stage[1] = c.NSTAGE > 1 ? take((size_t)c.STAGE) : stage[0];  // one stage: huge items (large T)
        stage[2] = c.NSTAGE > 2 ? take((size_t)c.STAGE) : stage[0];
        fw = take(sizeof(float) * (size_t)NM * (c.FT + T));
        dl = take(sizeof(float) * (size_t)NM * T);
        // the state-constant table only for the T < 40 kernels (no task splitting): at large T its
        // NM * T floats came out of the item stages and tipped dense C4 T = 80 batches into the
        // one-model-at-a-time retry (2.4x slower); those kernels compute the constant inline
        sc = take(T < 40 ? sizeof(float) * (size_t)NM * T : 0);
        ctl = take(1024);  // item descriptors and layouts, mbarriers, counters
        total = o;
    }
};


// Optional pipeline trace (HGM_TRACE=1): globaltimer stamps of CTA 0, one launch.
__device__ unsigned long long *g_trace = nullptr;
__device__ __forceinline__ void trace(int m, int ev) {
    if (blockIdx.x == 0 && g_trace && m < 64) {  // (CTA 0 only reads the pointer)
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_trace[m * 8 + ev] = t;
    }
}

// Control block in shared memory.
struct Ctl {
    WorkItem w[3];      // stage descriptors (w[s].live == 0: no more items)
    StageLayout lay[3]; // stage layouts
    int row_claim[3];   // next unconverted b row of the stage's item
    int task_claim[3];  // next unclaimed 32-task group
    uint64_t raw[3];    // stage inputs landed (copy-warp arrival + TMA bytes)
    uint64_t conv[3];   // every b row converted (one tx unit per row)
    uint64_t free_[3];  // stage released: one arrival per compute warp
};


// Issue the input copies of item (w, d) into stage s (producer lane 0): the alpha_{i+1}
// rows of the tile's b nodes straight into the candidate-entry area (the layer's state
// stride is the entry stride, so entry e = state slot qb0 - ppad + e), the direction
// rows, and the small ranges of the dummy-form slots, the unary row, the scene index.
template <int NM, bool kHasNext>
__device__ __forceinline__ void issue_stage(const SceneView &sc, WorkItem &w, const float *hist,
                                            int64_t L, int layer, const float *__restrict__ U, int64_t ui_off, int T,
                                            const SmemPlan &sp, unsigned char *smem, int s, uint64_t *bar,
                                            const unsigned char *__restrict__ book, unsigned book_bytes,
                                            bool dep_wait) {
    constexpr int EPF = entry_floats(NM);
    const InstDesc &d = w.d;
    const StageLayout ly = item_layout(w, T, NM, (int)book_bytes);
    unsigned char *sb = smem + sp.stage[s];
    Copier cl(bar);
    const int64_t nxo = (int64_t)(layer + 1) * L + d.off;  // alpha layer i+1 of this window (from the aligned base)
    const int Sw = d.we - d.wb;
    // step-independent inputs first (scene index, unary row, bookkeeping) ...
    w.th0 = w.qa - cl.range(sb + ly.th, sc.theta_pad, w.qa, w.qa1);  // TH[q] holds theta_pad[th0 + q]
    w.tb0 = cl.range(sb + ly.tb, sc.theta_pad, w.qb0, w.qb1);         // theta(b -> c) of the b rows' entries
    w.uc0 = cl.range(sb + ly.uc, U, ui_off + (int64_t)w.B0 * NM, ui_off + (int64_t)w.Cend * NM);
    w.tc0 = cl.range(sb + ly.tc, sc.t, w.B0, w.Cend);
    if (w.B1 > w.B0) cl.raw(sb + ly.ni, sc.ninfo + w.B0, (unsigned)(sizeof(int4) * (w.B1 - w.B0)));
    cl.raw(sb + ly.bk, book + (size_t)w.idx * book_bytes, book_bytes);  // the item's bookkeeping
    const int f_lo = max(0, w.F0 - T), f_hi = min(sc.fmax + 1, w.F1 + T);  // first_tab over [F0 - T, F1 + T]
    w.ft0 = cl.range(sb + ly.ftab, sc.ft, f_lo, f_hi + 1);
    w.flo = f_lo;
    // ... then the alpha layer i+1, which the previous step's grid writes: under programmatic
    // dependent launch the first item's static copies are in flight before this wait
    if (dep_wait) asm volatile("griddepcontrol.wait;" ::: "memory");
    if (kHasNext) {
        cl.range(sb + ly.en, hist, nxo + (int64_t)(w.qb0 - d.ppad) * EPF, nxo + (int64_t)(w.qb1 - d.ppad) * EPF);
        w.we0 = cl.range(sb + ly.we, hist, nxo + (int64_t)(d.ntail + w.B0 - d.wb) * EPF,
                         nxo + (int64_t)(d.ntail + w.Cend - d.wb) * EPF);
        w.eb0 = cl.range(sb + ly.eb, hist, nxo + (int64_t)(d.ntail + Sw + w.B0 - d.wb) * EPF,
                         nxo + (int64_t)(d.ntail + Sw + w.B1 - d.wb) * EPF);
        w.ee0 = cl.range(sb + ly.ee, hist, nxo + (int64_t)(d.ntail + 2 * Sw) * EPF,
                         nxo + (int64_t)(d.ntail + 2 * Sw + 1) * EPF);
    }
    cl.close();  // (the stage was released by the consumers' empty[s] arrivals, after their reads)
}

#ifndef HGM_KDP_MINB
#define HGM_KDP_MINB 2  // CTAs per SM the register allocation must allow (3 measured 11 % slower on C3)
#endif
template <int NM, bool kHasNext, bool kSplit>
__global__ void __launch_bounds__(KDP_BLOCK, HGM_KDP_MINB) k_dp_fused(SceneView sc, const WorkItem *__restrict__ items,
                                                             int nitems, int *__restrict__ counter,
                                                             float *__restrict__ hist, int64_t L, int layer,
                                                             int has_prev, StepConstB kc, const float *__restrict__ U,
                                                             int64_t ui_off, DPParams p, TileCaps caps,
                                                             const unsigned char *__restrict__ book) {
    constexpr int EPF = entry_floats(NM);
    extern __shared__ __align__(128) unsigned char smem[];
    const SmemPlan sp(caps, p.T, NM);
    const BookPlan bp(caps, p.T);
    const int nstage = caps.NSTAGE;  // 2 (double-buffered) or 1 (items too large for two)
    Ctl *ctl = reinterpret_cast<Ctl *>(smem + sp.ctl);
    float *DL = reinterpret_cast<float *>(smem + sp.dl);  // [T][NM] lambda2 |g_i - dt|
    float *fw = reinterpret_cast<float *>(smem + sp.fw);  // [FT + T][NM] frame minima of w
    const int T = p.T;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    float *SCG = reinterpret_cast<float *>(smem + sp.sc);  // [T][NM] lambda2 |g_{i-1} - g| (state constants)
    for (int q = tid; q < T * NM; q += KDP_THREADS) {
        const int dt = q / NM, k = q - dt * NM;
        DL[q] = delta_term(p.l2, kc.c[k].x, dt);
        if constexpr (!kSplit) SCG[q] = state_const(p.l2, kc.c[k].y, dt);
    }
    if (tid == 0) {
        for (int st = 0; st < 3; ++st) {
            mbar_init(&ctl->raw[st], 1);
            mbar_init(&ctl->conv[st], 1);
            mbar_init(&ctl->free_[st], KDP_WARPS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // PDL (launch_nm): let the next step's grid launch as our CTAs retire.  The copy warp is
    // the one that touches data of the previous step's grid (the alpha layer i+1 it
    // bulk-copies, the (eps, eps) slot that grid reset): it waits (griddepcontrol.wait) only
    // after claiming its first item and issuing that item's step-independent copies.  The
    // compute warps read nothing but the stages; they wait here too, which parks them in
    // hardware instead of polling the first stage's mbarrier while the previous grid runs.
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (warp < KDP_WARPS) asm volatile("griddepcontrol.wait;" ::: "memory");
    if (warp == KDP_WARPS) {
        // ---------------- copy warp: item m goes to stage m % 2 once item m-2 left it; it
        // also computes the dummy-form states (eps, b) and (eps, eps) of each item
        // lane 0 claims one item ahead: the claim and the descriptor load of item m+1 are in
        // flight while item m-1 still occupies the stage item m+1 will use
        int next_idx = lane == 0 ? atomicAdd(counter, 1) : 0;
        // st = m % nstage, use = m / nstage (how many items stage st held before), stepped
        // incrementally: nstage is a runtime value and an integer division costs ~20 instructions
        for (int m = 0, st = 0, use = 0;; ++m, st = (st + 1 == nstage) ? 0 : st + 1, use += st == 0 ? 1 : 0) {
            WorkItem pre{};
            if (lane == 0) {
                if (next_idx < nitems) pre = items[next_idx];
                next_idx = next_idx < nitems ? atomicAdd(counter, 1) : nitems;
            }
            if (use >= 1) mbar_wait(&ctl->free_[st], (use - 1) & 1, 1024);
            if (lane == 0) trace(m, 4);
            if (lane == 0) {
                WorkItem &nw = ctl->w[st];
                if (pre.live) {
                    nw = pre;
                    ctl->lay[st] = item_layout(nw, T, NM, (int)bp.total);
                    ctl->row_claim[st] = 0;
                    ctl->task_claim[st] = 0;
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&ctl->conv[st])),
                                 "r"((unsigned)(nw.B1 - nw.B0))
                                 : "memory");
                    issue_stage<NM, kHasNext>(sc, nw, hist, L, layer, U, ui_off, T, sp, smem, st, &ctl->raw[st], book,
                                              (unsigned)bp.total, m == 0);
                    trace(m, 5);
                } else {
                    nw.live = 0;
                    mbar_arrive(&ctl->raw[st]);
                }
            }
            if (m == 0) asm volatile("griddepcontrol.wait;" ::: "memory");  // (every lane: the dummy forms below)
            mbar_wait(&ctl->raw[st], use & 1);
            if (lane == 0) trace(m, 6);
            const WorkItem &w = ctl->w[st];
            if (!w.live) break;
            if (!w.primary) continue;  // another item of this b-tile finishes its dummy-form states
            const InstDesc &d = w.d;
            const StageLayout &ly = ctl->lay[st];
            const unsigned char *sb = smem + sp.stage[st];
            const float *UC = reinterpret_cast<const float *>(sb + ly.uc);
            const float *WE = reinterpret_cast<const float *>(sb + ly.we);
            const int4 *NI = reinterpret_cast<const int4 *>(sb + ly.ni);
            const float *EE = reinterpret_cast<const float *>(sb + ly.ee);
            const int *FTAB = reinterpret_cast<const int *>(sb + ly.ftab);
            auto first = [&](int f) { return f <= 0 ? 0 : (f > sc.fmax ? sc.S : FTAB[w.ft0 + (f - w.flo)]); };
            const int F0 = w.F0, F1 = w.F1, B0 = w.B0, NBr = w.B1 - w.B0, Sw = d.we - d.wb;
            const int wend = d.o + caps.W;
            float *cur = hist + (int64_t)layer * L + d.off;
            const int nfw = min(F1 + T - 1, wend) - F0;  // frames [F0, F1 + T - 1) inside the window
            for (int q = lane; q < nfw * NM; q += 32) {  // frame minima of w(c) = alpha_{i+1}(c, eps) + lambda1 U_i(c)
                const int fi = q / NM, k = q - fi * NM, f = F0 + fi;
                float wm = INFINITY;
                const int c1 = first(f + 1);
                for (int c = first(f); c < c1; ++c)
                    wm = fminf(wm, msg_n(kHasNext ? WE[w.we0 + (c - B0) * EPF + k] : 0.f, UC[w.uc0 + (c - B0) * NM + k]));
                fw[q] = wm;
            }
            __syncwarp();
            for (int q = lane; q < NBr * NM; q += 32) {  // (eps, b): frames (t'(b), t'(b) + T) in the window
                const int rb = q / NM, k = q - rb * NM;
                const int tb = NI[rb].x;
                float r = INFINITY;
                const int f1 = min(tb + T, wend);
                for (int f = tb + 1; f < f1; ++f) r = fminf(r, fw[(f - F0) * NM + k]);
                cur[(int64_t)(d.ntail + Sw + B0 + rb - d.wb) * EPF + k] =
                    fminf(r, __fadd_rn(p.l1W, kHasNext ? EE[w.ee0 + k] : 0.f));
            }
            if (lane < NM) {  // (eps, eps): this item's frames, min-reduced into the slot (reset to +inf by step i+1)
                float r = __fadd_rn(p.l1W, kHasNext ? EE[w.ee0 + lane] : 0.f);
                for (int f = F0; f < F1; ++f) r = fminf(r, fw[(f - F0) * NM + lane]);
                atomicMin(reinterpret_cast<unsigned *>(cur + (int64_t)(d.ntail + 2 * Sw) * EPF + lane), __float_as_uint(r));
                if (has_prev && F0 == d.o)  // the next step's slot starts at +inf
                    (cur - L)[(int64_t)(d.ntail + 2 * Sw) * EPF + lane] = INFINITY;
            }
            __syncwarp();
        }
        return;
    }
    for (int m = 0, s = 0, use = 0;; ++m, s = (s + 1 == nstage) ? 0 : s + 1, use += s == 0 ? 1 : 0) {
        if (tid == 0) trace(m, 0);
        mbar_wait(&ctl->raw[s], use & 1);
        if (tid == 0) trace(m, 1);
        const WorkItem &w = ctl->w[s];
        if (!w.live) break;
        const InstDesc &d = w.d;
        const StageLayout &ly = ctl->lay[s];
        unsigned char *sb = smem + sp.stage[s];
        float *b_ean = reinterpret_cast<float *>(sb + ly.bean);  // [NB][NM] lambda1 W^d + alpha_{i+1}(eps, b)
        const float *TH = reinterpret_cast<const float *>(sb + ly.th);
        const float *TB = reinterpret_cast<const float *>(sb + ly.tb);
        float *EN = reinterpret_cast<float *>(sb + ly.en);
        const float *UC = reinterpret_cast<const float *>(sb + ly.uc);
        const int *TC = reinterpret_cast<const int *>(sb + ly.tc);
        const int4 *NI = reinterpret_cast<const int4 *>(sb + ly.ni);
        const float *EB = reinterpret_cast<const float *>(sb + ly.eb);
        const int *FTAB = reinterpret_cast<const int *>(sb + ly.ftab);
        const int B0 = w.B0, B1 = w.B1, A0 = w.A0;
        const int NBr = B1 - B0;
        float *cur = hist + (int64_t)layer * L + d.off;
        auto first = [&](int f) { return f <= 0 ? 0 : (f > sc.fmax ? sc.S : FTAB[w.ft0 + (f - w.flo)]); };
        const unsigned char *bk = sb + ly.bk;  // the item's bookkeeping (k_item_prep)
        const int nst = *reinterpret_cast<const int *>(bk + bp.nst);
        const Seg *seg = reinterpret_cast<const Seg *>(bk + bp.seg);
        const int *r_ofs = reinterpret_cast<const int *>(bk + bp.rows);  // [NA] offset of row x in TH
        const int *r_en = r_ofs + caps.NA;  // entry index of row x's column 0 in EN
        const int *r_q = r_en + caps.NA;    // qstart[x] (compact band: coincidence flags)
        const int *r_qp = r_q + caps.NA;    // qpad[x] (padded band: alpha slots)
        const int *r_fc = r_qp + caps.NA;   // first / last coincident column
        const int *r_lc = r_fc + caps.NA;
        const uint8_t *smap = bk + bp.map;

        // ---- messages: warps claim b rows; each row's entries become messages in place and
        // its (b, eps) state is finished; every finished row completes one tx unit of conv[s]
        for (;;) {
            int rb = 0;
            if (lane == 0) rb = atomicAdd(&ctl->row_claim[s], 1);
            rb = __shfl_sync(0xffffffffu, rb, 0);
            if (rb >= NBr) break;
            const int4 ni = NI[rb];
            const int tb = ni.x, c0 = ni.y;
            const int len = min(first(tb + T), d.we) - c0;  // candidates of row b in this window (R1, R2)
            const int e0 = ni.w - w.qb0;
#ifdef HGM_DEBUG_CHECKS
            if (e0 < 0 || w.tb0 < 0 || w.tb0 > 3 || ly.total > caps.STAGE || e0 + len > w.qb1 - w.qb0 + 8 ||
                c0 < B0 || c0 > w.Cend || tb < w.F0 || tb >= w.F1) {
                if (lane == 0)
                    printf("conv: blk %d item F[%d,%d) G[%d,%d) A0 %d B0 %d B1 %d rb %d nA %d ni (%d,%d,%d,%d) qb0 %d qb1 %d "
                           "tb0 %d prim %d len %d lay.total %d STAGE %d tb %d\n",
                           blockIdx.x, w.F0, w.F1, w.G0, w.G1, A0, B0, B1, rb, w.nA, ni.x, ni.y, ni.z, ni.w, w.qb0, w.qb1,
                           w.tb0, w.primary, len, ly.total, caps.STAGE, ly.tb);
                continue;
            }
#endif
            float mn[NM];
#pragma unroll
            for (int k = 0; k < NM; ++k) mn[k] = INFINITY;
#pragma unroll 2
            for (int j = lane; j < len; j += 32) {
                const int e = e0 + j, cc = c0 + j - B0;
                const int dt = TC[w.tc0 + cc] - tb;
                float ent[EPF];
                if (kHasNext) ld_entry<EPF>(EN + (size_t)e * EPF, ent);  // alpha_{i+1}(c, b), landed by TMA
                const float *u = UC + w.uc0 + cc * NM;  // lambda1 U_i(c) (K-U's scaled table)
                const float *dl = DL + dt * NM;
                msg_build<NM, kHasNext>(ent, u, dl, mn);
                ent[NM] = TB[w.tb0 + e];  // theta(b -> c)
#pragma unroll
                for (int k = NM + 1; k < EPF; ++k) ent[k] = 0.f;
#pragma unroll
                for (int q = 0; q < EPF / 4; ++q)
                    reinterpret_cast<float4 *>(EN + (size_t)e * EPF)[q] =
                        make_float4(ent[4 * q], ent[4 * q + 1], ent[4 * q + 2], ent[4 * q + 3]);
            }
            float bm = INFINITY;
#pragma unroll
            for (int k = 0; k < NM; ++k) {  // n >= 0: float order = unsigned bit order
                const float v = __uint_as_float(__reduce_min_sync(0xffffffffu, __float_as_uint(mn[k])));
                if (lane == k) bm = v;
            }
            if (lane < NM) {
                const float ean = __fadd_rn(p.l1W, kHasNext ? EB[w.eb0 + rb * EPF + lane] : 0.f);
                b_ean[rb * NM + lane] = ean;  // lambda1 W^d + alpha_{i+1}(eps, b)
                if (w.primary) cur[(int64_t)(d.ntail + B0 + rb - d.wb) * EPF + lane] = fminf(bm, ean);  // (b, eps)
            }
            __syncwarp();
            // release: the row's shared-memory writes (messages, b_ean) happen-before the task
            // phase of every warp that acquires conv[s] (complete_tx itself is relaxed)
            if (lane == 0) {
                __threadfence_block();
                mbar_complete_tx(&ctl->conv[s], 1);
            }
        }
        mbar_wait(&ctl->conv[s], use & 1);  // all rows of the item are messages now
        // ---- P3: real states.  A lane task is one b with a PAIR of a's of the same a-frame
        // (same candidate range), so each candidate entry (b, c_j) is loaded once for two
        // states; warps claim 32-task groups (segments by descending trip count).  An item
        // with few tasks and long trips (large T: a few hundred states of hundreds of
        // candidates) would leave warps idle behind the one holding the last group, so there
        // LPT = 2..8 lanes share a task, each taking a contiguous share of its candidates, and
        // the shares' minima are combined by shuffles (min is exact and order-free: same bits).
        int lsh = 0;  // (a cost model that also split mid-size items measured 11-16 % slower on C4
                      // T = 40 / rho = 8: each share repeats the task decode and the combine)
        if constexpr (kSplit) {  // (a launch-time choice: compiled in, the split costs C3 1.9 %)
            if (nst > 0)  // seg[0]: the longest trip (descending order); shares of >= 48 candidates
                while (lsh < 3 && (nst << (lsh + 1)) <= 8 * KDP_THREADS && (seg[0].trip >> (lsh + 1)) >= 48) ++lsh;
        }
        const int LPT = 1 << lsh, sub = lane & (LPT - 1);
        for (;;) {
            int s0 = 0;
            if (lane == 0) s0 = atomicAdd(&ctl->task_claim[s], 32 >> lsh);
            s0 = __shfl_sync(0xffffffffu, s0, 0);
            if (s0 >= nst) break;
            const int st = s0 + (lane >> lsh);
            const bool live = st < nst;
            const Seg sg = seg[live ? smap[st] : smap[nst - 1]];
            int trip = 0, b = B0, a0 = A0;
            bool two = false;
            if (live) {
                const int r = st - sg.start;
                const int ci = sg.nb > 1 ? (int)__umulhi((unsigned)r, sg.inv) : r;
                b = sg.b0 + (r - ci * sg.nb);
                a0 = sg.a0 + 2 * ci;
                two = a0 + 1 < sg.f1a;
                trip = sg.trip;
            }
            const int a1 = two ? a0 + 1 : a0;
            const int ra0 = a0 - A0, ra1 = a1 - A0, rbt = w.nA + (b - B0);  // row-table rows (BookPlan)
            const int colb = b - sg.f1a;  // column of b in the rows of the a-frame
            const float *erow = EN + (size_t)r_en[rbt] * EPF;
            const float *arow0 = TH + r_ofs[ra0] + sg.aoff, *arow1 = TH + r_ofs[ra1] + sg.aoff;
            const float th_ab0 = live ? TH[r_ofs[ra0] + colb] : 0.f, th_ab1 = live ? TH[r_ofs[ra1] + colb] : 0.f;
            auto dirty_of = [&](int ra) {
                const int lca = r_lc[ra];
                return (lca >= 0 && lca >= min(colb, sg.aoff) && r_fc[ra] <= max(colb, sg.aoff + trip - 1));
            };
            const bool dirty = live && (dirty_of(ra0) || dirty_of(ra1) || r_fc[rbt] < trip);
            float R0[NM], R1[NM];
#pragma unroll
            for (int k = 0; k < NM; ++k) R0[k] = R1[k] = INFINITY;
            const int per = (trip + LPT - 1) >> lsh;  // this lane's share [jb, je) of the candidates
            const int jb = min(trip, sub * per), je = min(trip, jb + per);
            if (!__any_sync(0xffffffffu, dirty)) {
                task_loop<NM, EPF>(erow + (size_t)jb * EPF, arow0 + jb, arow1 + jb, th_ab0, th_ab1, je - jb, kc, p.l23,
                                   R0, R1);
            } else {  // exact flag-aware loop (coincident points, R10): the padded band holds NaN
                      // for the direction of a zero-length ray, so the flags come with the angles
                const bool co_ab0 = live && isnan(th_ab0);
                const bool co_ab1 = live && isnan(th_ab1);
                for (int j = jb; j < je; ++j) {
                    float e0[EPF];
                    ld_entry<EPF>(erow + (size_t)j * EPF, e0);
                    const bool cbc = isnan(e0[NM]);
                    const bool cac0 = isnan(arow0[j]);
                    const bool cac1 = isnan(arow1[j]);
#pragma unroll
                    for (int k = 0; k < NM; ++k) {
                        R0[k] = fminf(R0[k], cand_value(e0[k], e0[NM], th_ab0, arow0[j], cbc || co_ab0, cbc || cac0,
                                                        kc.c[k].z, kc.c[k].w, p.l23));
                        R1[k] = fminf(R1[k], cand_value(e0[k], e0[NM], th_ab1, arow1[j], cbc || co_ab1, cbc || cac1,
                                                        kc.c[k].z, kc.c[k].w, p.l23));
                    }
                }
            }
            for (int o = 1; o < LPT; o <<= 1) {  // combine the shares (the lanes of a task are adjacent)
#pragma unroll
                for (int k = 0; k < NM; ++k) {
                    R0[k] = fminf(R0[k], __shfl_xor_sync(0xffffffffu, R0[k], o));
                    R1[k] = fminf(R1[k], __shfl_xor_sync(0xffffffffu, R1[k], o));
                }
            }
            HGM_DCHECK(!live || (ra0 >= 0 && ra1 < w.nA + NBr && rbt < w.nA + NBr && r_qp[ra0] + colb >= d.ppad &&
                                 r_qp[ra1] + colb < d.ppad + d.npp && r_en[rbt] + trip <= w.qb1 - w.qb0 + 8));
            if (live && sub == 0) {
                float out0[EPF], out1[EPF];
#pragma unroll
                for (int k = 0; k < NM; ++k) {
                    float sc_g;  // state_const(l2, g_{i-1}, g): same gap for both states
                    if constexpr (!kSplit) sc_g = SCG[sg.g * NM + k];
                    else sc_g = state_const(p.l2, kc.c[k].y, sg.g);
                    const float ean = b_ean[(b - B0) * NM + k];
                    out0[k] = fminf(__fadd_rn(R0[k], sc_g), ean);
                    out1[k] = fminf(__fadd_rn(R1[k], sc_g), ean);
                }
#pragma unroll
                for (int k = NM; k < EPF; ++k) out0[k] = out1[k] = 0.f;
                float4 *dst0 = reinterpret_cast<float4 *>(cur + (int64_t)(r_qp[ra0] + colb - d.ppad) * EPF);
#pragma unroll
                for (int q = 0; q < EPF / 4; ++q)
                    dst0[q] = make_float4(out0[4 * q], out0[4 * q + 1], out0[4 * q + 2], out0[4 * q + 3]);
                if (two) {
                    float4 *dst1 = reinterpret_cast<float4 *>(cur + (int64_t)(r_qp[ra1] + colb - d.ppad) * EPF);
#pragma unroll
                    for (int q = 0; q < EPF / 4; ++q)
                        dst1[q] = make_float4(out1[4 * q], out1[4 * q + 1], out1[4 * q + 2], out1[4 * q + 3]);
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&ctl->free_[s]);  // this warp is done with stage s
        if (tid == 0) trace(m, 3);
    }
}

// (eps, eps) slots of the first layer of a chunk start at +inf (later layers: reset by K-DP)
__global__ void k_init_ee(const InstDesc *__restrict__ inst, int ninst, float *__restrict__ hist, int64_t L,
                          int layer, int NM) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= ninst * NM) return;
    const int k = q / NM, m = q - k * NM;
    const InstDesc d = inst[k];
    hist[(int64_t)layer * L + d.off + (int64_t)(d.ntail + 2 * (d.we - d.wb)) * entry_floats(NM) + m] = INFINITY;
}

// Work items of a chunk, one thread per window: for every global b-tile meeting the
// window's frames, its a-frame chunks (one chunk unless T is large) that meet them,
// clipped; the first item of each b-tile is its "primary".  Written at
// item_base[k] - base0 ...; descriptors are valid for every step of the chunk.
__global__ void k_items(SceneView sc, const InstDesc *__restrict__ inst, int ninst, int W, int T,
                        const int32_t *__restrict__ gstart, const int32_t *__restrict__ tile_of, int tf_lo,
                        const int32_t *__restrict__ sub_begin, const int32_t *__restrict__ sub_g,
                        const int32_t *__restrict__ item_base, int base0, WorkItem *items) {
    // one warp per window; lane j of a round takes b-tile g_first + round*32 + j (a window
    // of the single-instance regime has hundreds of tiles and thousands of chunks)
    const int k = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
    if (k >= ninst) return;
    const InstDesc d = inst[k];
    const int g_first = __ldg(tile_of + (d.o - tf_lo)), g_last = __ldg(tile_of + (d.o + W - 1 - tf_lo));
    int idx0 = __ldg(item_base + k) - base0;
    for (int g0 = g_first; g0 <= g_last; g0 += 32) {
        const int gt = g0 + lane;
        const bool on = gt <= g_last;
        int F0 = 0, F1 = 0, sb0 = 0, sb1 = 0, n = 0;
        if (on) {
            F0 = max(__ldg(gstart + gt), d.o);
            F1 = min(__ldg(gstart + gt + 1), d.o + W);
            sb0 = __ldg(sub_begin + gt);
            sb1 = __ldg(sub_begin + gt + 1);
            for (int sb = sb0; sb < sb1; ++sb)  // chunks meeting the window (the first always counts)
                n += (sb == sb0 || max(__ldg(sub_g + 2 * sb), d.o) < min(__ldg(sub_g + 2 * sb + 1), F1)) ? 1 : 0;
        }
        const int incl = warp_incl_scan(n, lane);
        int idx = idx0 + incl - n;
        idx0 += __shfl_sync(0xffffffffu, incl, 31);
        if (!on) continue;
        bool first_of_tile = true;
        for (int sb = sb0; sb < sb1; ++sb) {
            WorkItem w{};
            w.d = d;
            w.live = 1;
            w.F0 = F0;
            w.F1 = F1;
            w.G0 = max(__ldg(sub_g + 2 * sb), d.o);
            w.G1 = min(__ldg(sub_g + 2 * sb + 1), w.F1);
            if (w.G0 >= w.G1 && !first_of_tile) continue;  // chunk entirely before the window
            w.primary = first_of_tile ? 1 : 0;
            first_of_tile = false;
            w.idx = idx;
            w.B0 = sc.first(w.F0);
            w.B1 = sc.first(w.F1);
            w.A0 = max(sc.first(w.G0), d.wb);
            w.Cend = min(sc.first(w.F1 + T - 1), d.we);
            w.qa = __ldg(sc.qpad + w.A0);
            w.qa1 = __ldg(sc.qpad + max(sc.first(w.G1), w.A0));
            w.nA = min(max(sc.first(w.G1), w.A0), w.B0) - w.A0;
            w.qb0 = __ldg(sc.qpad + w.B0);
            w.qb1 = __ldg(sc.qpad + w.B1);
            items[idx++] = w;
        }
    }
}

// Step-independent bookkeeping of every work item of a chunk (one CTA per item):
// the segment table of its real states (a (b-frame, a-frame) segment shares its
// candidate range [minnode(t'(b)+1), minnode(t'(a)+T))) in
// descending trip order with prefix starts, the state -> segment map, and the row tables.
__global__ void __launch_bounds__(256) k_item_prep(SceneView sc, const WorkItem *__restrict__ items, TileCaps caps,
                                                   int T, unsigned char *__restrict__ book) {
    const BookPlan bp(caps, T);
    const WorkItem w = items[blockIdx.x];
    unsigned char *bk = book + (size_t)blockIdx.x * bp.total;
    Seg *seg = reinterpret_cast<Seg *>(bk + bp.seg);
    int *r_ofs = reinterpret_cast<int *>(bk + bp.rows);
    int *r_en = r_ofs + caps.NA, *r_q = r_en + caps.NA, *r_qp = r_q + caps.NA, *r_fc = r_qp + caps.NA,
        *r_lc = r_fc + caps.NA;
    uint8_t *smap = bk + bp.map;
    __shared__ int s_cnt[256];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // segments (b-frame f, gap g) whose a-frame f - g lies in the item's chunk [G0, G1):
    // gaps [gmin, gmax]; the host keeps (F1 - F0) * (gmax - gmin + 1) <= 255 (uint8 map)
    const int F0 = w.F0, F1 = w.F1;
    const int gmin = max(1, F0 - w.G1 + 1), gmax = min(T - 1, F1 - 1 - w.G0);
    const int nseg = max(0, (F1 - F0) * (gmax - gmin + 1));
    const int th0 = w.qa & ~3;  // theta_pad index the stage's TH[0] holds (the copy starts 16-byte aligned)
    for (int r = tid; r < w.nA + (w.B1 - w.B0); r += blockDim.x) {
        const int x = r < w.nA ? w.A0 + r : w.B0 + (r - w.nA);  // the a rows before B0, then the b rows
        const int4 ni = __ldg(sc.ninfo + x);  // (t', minnode(t'+1), qstart, qpad)
        r_ofs[r] = ni.w - th0;
        r_en[r] = ni.w - w.qb0;
        r_q[r] = ni.z;
        r_qp[r] = ni.w;
        r_fc[r] = __ldg(sc.rfc + x);  // whole (unclipped) row: conservative
        r_lc[r] = __ldg(sc.rlc + x);
    }
    __shared__ int s_key[256];
    Seg sg{};
    int cnt = 0;
    if (tid < nseg) {  // segments (enumerated gap-major), then ordered by candidate count below
        const int g = gmin + tid / (F1 - F0);
        const int f = F0 + tid % (F1 - F0);
        if (f - g >= w.d.o && f - g >= w.G0 && f - g < w.G1) {
            sg.g = g;
            sg.b0 = sc.first(f);
            sg.nb = sc.first(f + 1) - sg.b0;
            sg.a0 = sc.first(f - g);
            sg.f1a = sc.first(f - g + 1);
            const int c0 = sc.first(f + 1);
            sg.trip = max(0, min(sc.first(f - g + T), w.d.we) - c0);
            sg.aoff = c0 - sg.f1a;
            sg.inv = sg.nb > 1 ? 0xffffffffu / (unsigned)sg.nb + 1u : 0u;  // ceil(2^32 / nb)
            cnt = sg.nb * ((sg.f1a - sg.a0 + 1) >> 1);  // lane tasks: one b, a pair of a's
        }
    }
    // rank = position in descending trip order (ties: enumeration order), so the 32 lanes of
    // a task group see near-equal trip counts (warp lanes idle less at the end of the loop)
    s_key[tid] = (tid < nseg && cnt > 0) ? sg.trip : -1;
    __syncthreads();
    int rank = 0;
    if (tid < nseg) {
        const int key = s_key[tid];
        for (int j = 0; j < nseg; ++j) {
            const int kj = s_key[j];
            rank += (kj > key || (kj == key && j < tid)) ? 1 : 0;
        }
    }
    if (tid < nseg) s_cnt[rank] = cnt;
    __syncthreads();
    if (warp == 0) {  // prefix over the segments (nseg <= 255)
        int carry = 0;
        for (int r0 = 0; r0 < nseg; r0 += 32) {
            const int v = r0 + lane < nseg ? s_cnt[r0 + lane] : 0;
            const int incl = warp_incl_scan(v, lane);
            if (r0 + lane < nseg) s_cnt[r0 + lane] = carry + incl - v;
            carry += __shfl_sync(0xffffffffu, incl, 31);
        }
        if (lane == 0) *reinterpret_cast<int *>(bk + bp.nst) = carry;
    }
    __syncthreads();
    if (tid < nseg) {
        sg.start = s_cnt[rank];
        seg[rank] = sg;
        for (int q = 0; q < cnt; ++q) smap[sg.start + q] = (uint8_t)rank;
    }
}

hgm_status launch_item_prep(const SceneView &v, const WorkItem *items, int nitems, const TileCaps &caps, int T,
                            unsigned char *book, cudaStream_t s) {
    if (nitems > 0) k_item_prep<<<nitems, 256, 0, s>>>(v, items, caps, T, book);
    return HGM_OK;
}

size_t item_book_bytes(const TileCaps &caps, int T) { return BookPlan(caps, T).total; }

// stage bytes of an item of the given sizes (host tiling; the layout the kernel uses)
size_t item_stage_bytes(int NE, int NTH, int NC, int NA, int NB, int FT, int T, int NM, int book) {
    return (size_t)StageLayout(NE, NTH, NC, NA, NB, FT, T, NM, book).total;
}

// ------------------------------------------------------------------ launchers
size_t dp_batch_smem(const TileCaps &c, int T, int NM) { return SmemPlan(c, T, NM).total; }

template <int NM>
static hgm_status launch_nm(const SceneView &v, const WorkItem *items, int nitems, const unsigned char *book,
                            int *counter, float *hist, int64_t L, int layer, bool has_next, bool has_prev,
                            const StepConstB &kc, const float *U, int64_t ui_off, const DPParams &p,
                            const TileCaps &caps, cudaStream_t s, bool pdl_ok) {
    const size_t smem = dp_batch_smem(caps, p.T, NM);
    // task splitting (kSplit) only where trips can be long enough to split (T >= 40)
    const bool split = p.T >= 40;
    auto kern = split ? (has_next ? k_dp_fused<NM, true, true> : k_dp_fused<NM, false, true>)
                      : (has_next ? k_dp_fused<NM, true, false> : k_dp_fused<NM, false, false>);
    int dev = 0;
    HGM_CUDA(cudaGetDevice(&dev));
    // the shared-memory attribute applies per device context: cache it per device (and the
    // occupancy it gives), under a lock -- calls on different devices / threads may race here
    static std::mutex mu;
    static int configured[64][4], occ[64][4], nsm_of[64];
    int bps = 1, nsm = 0;
    {
        std::lock_guard<std::mutex> lk(mu);
        const int d = dev < 0 || dev >= 64 ? 0 : dev, h = (has_next ? 1 : 0) + (split ? 2 : 0);
        if (dev < 0 || dev >= 64 || (int)smem > configured[d][h] || !nsm_of[d]) {
            HGM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            int b = 0;
            HGM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, KDP_BLOCK, smem));
            HGM_CUDA(cudaDeviceGetAttribute(&nsm_of[d], cudaDevAttrMultiProcessorCount, dev));
            if (dev >= 0 && dev < 64) {
                configured[d][h] = (int)smem;
                occ[d][h] = b;
            }
            bps = b;
        } else {
            bps = occ[d][h];
        }
        nsm = nsm_of[d];
    }
    const int grid = std::max(1, std::min(nitems, std::max(1, bps) * nsm));
    static int traced = 0;
    unsigned long long *tbuf = nullptr;
    static const bool trace_env = getenv("HGM_TRACE") != nullptr;  // (read once: this runs per launch)
    if (trace_env && !traced && layer == 10) {
        traced = 1;
        cudaMalloc(&tbuf, 64 * 8 * 8);
        cudaMemset(tbuf, 0, 64 * 8 * 8);
        cudaMemcpyToSymbol(g_trace, &tbuf, sizeof(tbuf));
    }
    // Programmatic dependent launch: the CTAs of this step may become resident as soon as
    // the previous step's CTAs retire (each triggers at its start), run their prologue (Delta
    // table, mbarriers) and then wait in griddepcontrol.wait until the previous step's grid
    // has completed and its alpha layer is visible -- the launch gap and the prologue leave
    // the per-step critical path (many short steps: single instances, few-window chunks).
    static const bool pdl_env = !(getenv("HGM_PDL") && atoi(getenv("HGM_PDL")) == 0);  // HGM_PDL=0: off (A/B)
    const bool pdl = pdl_env && pdl_ok;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(KDP_BLOCK);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    HGM_CUDA(cudaLaunchKernelEx(&cfg, kern, v, items, nitems, counter, hist, L, layer, has_prev ? 1 : 0, kc, U, ui_off,
                                p, caps, book));
    if (tbuf) {
        unsigned long long h[64 * 8], *z = nullptr;
        cudaMemcpy(h, tbuf, sizeof(h), cudaMemcpyDeviceToHost);
        cudaMemcpyToSymbol(g_trace, &z, sizeof(z));
        cudaFree(tbuf);
        unsigned long long t0 = h[0];
        fprintf(stderr, "HGM_TRACE grid=%d smem=%zu  (us since start) P:emptywait,issued,synced,raw,converted  C:wait,got,done\n",
                grid, smem);
        for (int m = 0; m < 64; ++m) {
            fprintf(stderr, "%2d", m);
            for (int e = 0; e < 8; ++e) fprintf(stderr, " %8.2f", h[m * 8 + e] ? (h[m * 8 + e] - t0) * 1e-3 : -1.0);
            fprintf(stderr, "\n");
        }
    }
    return HGM_OK;
}

hgm_status launch_dp_batch(int NM, const SceneView &v, const WorkItem *items, int nitems, const unsigned char *book,
                           int *counter, float *hist, int64_t L, int layer, bool has_next, bool has_prev,
                           const StepConstB &kc, const float *U, int64_t ui_off, const DPParams &p,
                           const TileCaps &caps, cudaStream_t s, bool pdl_ok) {
#define HGM_NM_CASE(n)                                                                                             \
    case n:                                                                                                        \
        return launch_nm<n>(v, items, nitems, book, counter, hist, L, layer, has_next, has_prev, kc, U, ui_off, p, \
                            caps, s, pdl_ok)
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
                        const int32_t *tile_of, int tf_lo, const int32_t *sub_begin, const int32_t *sub_g,
                        const int32_t *item_base, int base0, WorkItem *items, cudaStream_t s) {
    if (ninst > 0)
        k_items<<<(unsigned)((ninst + 3) / 4), 128, 0, s>>>(v, dinst, ninst, W, T, gstart, tile_of, tf_lo, sub_begin,
                                                            sub_g, item_base, base0, items);
    return HGM_OK;
}

hgm_status launch_init_ee(const InstDesc *dinst, int ninst, float *hist, int64_t L, int layer, int NM,
                          cudaStream_t s) {
    const int n = ninst * NM;
    if (n > 0) k_init_ee<<<(n + 255) / 256, 256, 0, s>>>(dinst, ninst, hist, L, layer, NM);
    return HGM_OK;
}

}  // namespace hgm
