// dp_window.cu -- K-DPW: the WHOLE recursion of PAPER.md Eqs. 10-11 (steps i = M..3) for
// one window x one batch of NM models of equal M, in ONE CTA, with the window's trellis
// resident in shared memory for all M-2 steps.
//
// Why: when a call has few windows (one model against one clip, C1; 50 models against
// 60-frame blocks; one model against a whole 754-node video at T = 10; a streaming push)
// the per-step kernel (dp_batch.cu: one launch per step, alpha layers through HBM) is
// bound by launch latency and per-step pipeline fill, not by arithmetic -- the paper's own
// launch-bound regime (one launch per step with a CPU sync; S = 60 blocks gave
// identical times on three GPUs).  Its remedy was a work-group that keeps the
// alpha row in local memory; here a CTA keeps a whole window:
//   TH   [npp]            directions theta(a -> c) of the window's padded band rows (static)
//   LAY  [(npp+2Sw+1)NM]  alpha layer: alpha_{i+1} at the start of step i, alpha_i at its end
//                         (pair states in padded band order, then (b,eps), (eps,a), (eps,eps))
//   ENT  [npp][EPF]       per candidate entry (b, c): the NM messages
//                         m(b,c) = alpha_{i+1}(c,b) + lambda1 U_i(c) + lambda2 |g_i - (t'c - t'b)|
//                         and theta(b -> c)
//   UR   [Sw][NM]         the unary row U_i of the window (TMA bulk copy, prefetched a step ahead)
//   node tables, the frame -> node table of the window, and the gap-major task list.
// Per step: phase 1 builds the messages, the (b,eps) row minima and the dummy-form terms
// from LAY (one warp per b row); phase 2 evaluates the real states (tasks claimed by warps:
// a task = one b with a PAIR of a's of one frame, so each entry load serves two states;
// longest candidate ranges first) and the dummy forms into LAY; one thread then streams
// LAY to the alpha history in HBM with a single TMA bulk store (cp.async.bulk), which
// overlaps the next step.  K-BT (backtrack.cu) re-evaluates its path from that history.
//
// The arithmetic is hgm_device.cuh's through dp_kdp.cuh's packed body (bit-identical to
// the per-state v0 kernel and to dp_batch.cu), so the backtrack stays exact.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "dp_kdp.cuh"

namespace hgm {

// 256, 512 or 1024 threads per CTA (launch_nm_w: ~32 warps per SM)
constexpr int KW_THREADS_MAX = 1024;

struct WinPlan {  // shared-memory plan (byte offsets), sized by the launch's maxima
    size_t th, ent, lay, ur, dn, wc, bean, nt, nlo, nhi, nro, nfc, nlc, ftl, task, dl, kc, kca, ctl, total;
    int lay_floats;
    __host__ __device__ WinPlan(const WinCaps &c, int NM) {
        size_t o = 0;
        auto take = [&](size_t bytes) {
            const size_t r = o;
            o = align16(o + bytes);
            return r;
        };
        lay_floats = (int)(((size_t)(c.NPP + 2 * c.SW + 1) * NM + 3) & ~(size_t)3);
        th = take(4 * (size_t)c.NPP);
        ent = take(4 * (size_t)went_floats(NM) * c.NPP);
        lay = take(4 * (size_t)lay_floats);
        ur = take(4 * ((size_t)NM * c.SW + 8));
        dn = take(4 * (size_t)NM * (2 * c.SW + 1));
        wc = take(NM >= 3 ? 4 * (size_t)NM * c.SW : 0);
        bean = take(4 * (size_t)NM * c.SW);
        nt = take(4 * (size_t)c.SW);
        nlo = take(4 * (size_t)c.SW);
        nhi = take(4 * (size_t)c.SW);
        nro = take(4 * (size_t)c.SW);
        nfc = take(4 * (size_t)c.SW);
        nlc = take(4 * (size_t)c.SW);
        ftl = take(4 * (size_t)(c.W + 2));
        task = take(4 * (size_t)c.NTASK);
        dl = take(4 * (size_t)c.T * NM);
        kc = take(sizeof(StepConstB));
        kca = take(16 * (size_t)c.M * NM);   // step constants of every step (float4 per model)
        ctl = take(48 + 4 * (KW_THREADS_MAX / 32 + 1));
        total = o;
    }
};

// CTA-wide exclusive scan of one int per thread; returns the prefix, *total the sum
template <int KW_WARPS>
__device__ __forceinline__ int cta_excl_scan(int v, int *s_warp, int *total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int incl = warp_incl_scan(v, lane);
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        const int w = lane < KW_WARPS ? s_warp[lane] : 0;
        const int wi = warp_incl_scan(w, lane);
        if (lane < KW_WARPS) s_warp[lane] = wi - w;
        if (lane == KW_WARPS - 1) s_warp[KW_WARPS] = wi;
    }
    __syncthreads();
    const int r = s_warp[warp] + incl - v;
    *total = s_warp[KW_WARPS];
    __syncthreads();
    return r;
}

// Optional step trace (HGM_TRACE_W=1, diagnosis): globaltimer stamps of CTA 0 at the
// phase boundaries of every step of one launch: [step][0..5]
__device__ unsigned long long *g_wtrace = nullptr;
// (the pointer is read ONCE per kernel, by thread 0 of CTA 0: a global load per call site
// stalled every step -- ncu attributed 9 % of K-DPW's stall samples to it)
__device__ __forceinline__ void wtrace(unsigned long long *wt, int s, int ev) {
    if (wt && s < 256) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        wt[s * 8 + ev] = t;
    }
}

template <int NM, int KW_THREADS>
__global__ void __launch_bounds__(KW_THREADS) k_dp_window(SceneView sc, const InstDesc *__restrict__ inst,
                                                           float *__restrict__ hist, int64_t L, int M,
                                                           WinStepPtrs sp, const float *__restrict__ U, int64_t nn,
                                                           int64_t n_lo, DPParams p, WinCaps caps,
                                                           const WinPlan pl) {
    constexpr int EPF = went_floats(NM);
    constexpr int KW_WARPS = KW_THREADS / 32;
    // the (eps, x) dummy forms: in the row warps' pass (one more reduction per model and row)
    // for small batches, else per (x, model) thread after the barrier from a per-node w table
    constexpr bool kMergeDummy = NM <= 2;
    extern __shared__ __align__(128) unsigned char smem[];
    // (the shared-memory plan comes in the parameter space, computed on the host: built
    // here, its offsets were rematerialised inside the loops -- ~4 % of the instructions)
    float *TH = reinterpret_cast<float *>(smem + pl.th);
    float *ENT = reinterpret_cast<float *>(smem + pl.ent);
    float *LAY = reinterpret_cast<float *>(smem + pl.lay);
    float *UR = reinterpret_cast<float *>(smem + pl.ur);
    float *DN = reinterpret_cast<float *>(smem + pl.dn);      // new dummy-form slots of the step
    float *WC = reinterpret_cast<float *>(smem + pl.wc);      // w(c) per node (NM >= 3)
    float *BEAN = reinterpret_cast<float *>(smem + pl.bean);
    int *NT = reinterpret_cast<int *>(smem + pl.nt);
    int *NLO = reinterpret_cast<int *>(smem + pl.nlo);
    int *NHI = reinterpret_cast<int *>(smem + pl.nhi);
    int *NRO = reinterpret_cast<int *>(smem + pl.nro);
    int *NFC = reinterpret_cast<int *>(smem + pl.nfc);
    int *NLC = reinterpret_cast<int *>(smem + pl.nlc);
    int *FTL = reinterpret_cast<int *>(smem + pl.ftl);
    unsigned *TASK = reinterpret_cast<unsigned *>(smem + pl.task);
    float *DL = reinterpret_cast<float *>(smem + pl.dl);
    StepConstB *s_kc = reinterpret_cast<StepConstB *>(smem + pl.kc);
    float4 *KCA = reinterpret_cast<float4 *>(smem + pl.kca);            // [M][NM] (g_i, g_{i-1}, A1, K2)
    uint64_t *ubar = reinterpret_cast<uint64_t *>(smem + pl.ctl);
    int *s_claim = reinterpret_cast<int *>(smem + pl.ctl + 8);
    int *s_ntask = reinterpret_cast<int *>(smem + pl.ctl + 12);
    float *EEN = reinterpret_cast<float *>(smem + pl.ctl + 16);   // [NM] lambda1 W^d + alpha_{i+1}(eps, eps)
    int *s_warp = reinterpret_cast<int *>(smem + pl.ctl + 48);    // KW_WARPS + 1 ints

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    unsigned long long *const wt = (blockIdx.x == 0 && tid == 0) ? g_wtrace : nullptr;
    const InstDesc d = inst[blockIdx.x];
    const int wb = d.wb, Sw = d.we - d.wb, npp = d.npp, T = p.T, o = d.o, W = caps.W;
    const int EE = npp + 2 * Sw;  // (eps, eps) slot
    const unsigned lay_bytes = (unsigned)(4 * (((size_t)(EE + 1) * NM + 3) & ~(size_t)3));
    const int nsteps = M - 2;

    if (tid == 0) {
        mbar_init(ubar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // the unary row of the first step (i = M - 1) streams in while the tables are built
    auto issue_u = [&](int i) {
        Copier cl(ubar);
        cl.range(UR, U, ((int64_t)i * nn + (wb - n_lo)) * NM, ((int64_t)i * nn + (wb - n_lo) + Sw) * NM);
        cl.close();
    };
    if (tid == 0) issue_u(M - 1);

    // ---- window tables (once): node info, frame -> node, direction rows
    for (int x = tid; x < Sw; x += KW_THREADS) {
        const int4 ni = __ldg(sc.ninfo + wb + x);  // (t', minnode(t'+1), qstart, qpad)
        NT[x] = ni.x;
        NLO[x] = min(ni.y, d.we) - wb;
        NHI[x] = min(sc.first(ni.x + T), d.we) - wb;
        NRO[x] = ni.w - d.ppad;
        NFC[x] = __ldg(sc.rfc + wb + x);
        NLC[x] = __ldg(sc.rlc + wb + x);
    }
    for (int f = tid; f <= W; f += KW_THREADS) FTL[f] = min(max(sc.first(o + f), wb), d.we) - wb;
    for (int q = tid; q < npp; q += KW_THREADS) TH[q] = __ldg(sc.theta_pad + d.ppad + q);
    for (int q = tid; q < M * NM; q += KW_THREADS) KCA[q] = __ldg(sp.step[q % NM] + q / NM);
    __syncthreads();
    // ---- task list (once): gap-major (longest candidate ranges first), per b-frame
    // segment (b, pair of a's of frame t'(b) - g): packed b | a0 << 16 | two << 31
    {
        int base = 0;
        for (int g = 1; g < T; ++g) {
            for (int b0 = 0; b0 < Sw; b0 += KW_THREADS) {
                const int b = b0 + tid;
                int na = 0, a_lo = 0;
                if (b < Sw) {
                    const int fa = NT[b] - g - o;
                    if (fa >= 0) {
                        a_lo = FTL[fa];
                        na = FTL[fa + 1] - a_lo;
                    }
                }
                const int nt = (na + 1) >> 1;
                int tot;
                const int at = base + cta_excl_scan<KW_WARPS>(nt, s_warp, &tot);
                HGM_DCHECK(at + nt <= caps.NTASK);
                for (int q = 0; q < nt; ++q) {
                    const int a0 = a_lo + 2 * q;
                    TASK[at + q] = (unsigned)b | ((unsigned)a0 << 16) | (a0 + 1 < a_lo + na ? 0x80000000u : 0u);
                }
                base += tot;
            }
        }
        if (tid == 0) *s_ntask = base;
        // ---- tasks in descending order of their candidate counts (a counting sort by trip,
        // once per window): the 32 lanes of a claimed group then run near-equal trips (the
        // gap-major order leaves Poisson-spread trips in a group, and the loop runs as long
        // as its longest lane).  Scratch: the entry area ENT, unused until the first step.
        // Order within a trip is arbitrary: every task owns its states, so no result changes.
        int *HIST = reinterpret_cast<int *>(ENT);                 // [Sw + 1] counts, then cursors
        unsigned *TMP = reinterpret_cast<unsigned *>(ENT) + ((Sw + 4) & ~3);  // [ntask]
        if ((size_t)((Sw + 4) & ~3) + (size_t)base <= (size_t)EPF * caps.NPP) {
            auto trip_of = [&](unsigned tk) {
                const int b = (int)(tk & 0xffffu), a0 = (int)((tk >> 16) & 0x7fffu);
                return min(Sw, max(0, NHI[a0] - NLO[b]));
            };
            for (int q = tid; q <= Sw; q += KW_THREADS) HIST[q] = 0;
            __syncthreads();
            for (int q = tid; q < base; q += KW_THREADS) {
                const unsigned tk = TASK[q];
                TMP[q] = tk;
                atomicAdd(&HIST[trip_of(tk)], 1);
            }
            __syncthreads();
            int carry = 0;  // first position of trip v = the tasks of trips > v
            for (int r0 = 0; r0 <= Sw; r0 += KW_THREADS) {
                const int r = r0 + tid, v = Sw - r;
                const int cnt = r <= Sw ? HIST[v] : 0;
                int tot;
                const int ex = cta_excl_scan<KW_WARPS>(cnt, s_warp, &tot);
                if (r <= Sw) HIST[v] = carry + ex;
                carry += tot;
            }
            __syncthreads();
            for (int q = tid; q < base; q += KW_THREADS) {
                const unsigned tk = TMP[q];
                TASK[atomicAdd(&HIST[trip_of(tk)], 1)] = tk;
            }
            __syncthreads();
        }
    }

    int u_use = 0;
    for (int s = 0; s < nsteps; ++s) {
        const int i = M - 1 - s;  // 0-based model node of this step; layer i - 2
        const bool has_next = s > 0;
        wtrace(wt, s, 0);
        // ---- step constants (model gaps / angles) and the Delta table
        if (tid == 0) {
            StepConstB kc{};
            for (int k = 0; k < NM; ++k) kc.c[k] = KCA[i * NM + k];
            for (int q = 0; q < (NM + 1) / 2; ++q) {
                const int k1 = min(2 * q + 1, NM - 1);
                kc.nA1[q] = make_float2(-kc.c[2 * q].z, -kc.c[k1].z);
                kc.nK2[q] = make_float2(-kc.c[2 * q].w, -kc.c[k1].w);
            }
            *s_kc = kc;
            *s_claim = 0;
        }
        for (int q = tid; q < T * NM; q += KW_THREADS) {
            const int dt = q / NM, k = q - dt * NM;
            DL[q] = delta_term(p.l2, KCA[i * NM + k].x, dt);
        }
        // the new dummy-form slots (DN: (x, eps) | (eps, x) | (eps, eps)) are built apart from
        // LAY (whose old ones phase 1 still reads); (eps, eps) starts at lambda1 W^d + its old
        // value and is min-reduced by phase 1
        if (tid < NM) {
            const float een = __fadd_rn(p.l1W, has_next ? LAY[EE * NM + tid] : 0.f);
            EEN[tid] = een;
            DN[2 * Sw * NM + tid] = een;
        }
        mbar_wait(ubar, u_use & 1);  // U_i landed
        ++u_use;
        const float *Ui = UR + (((int64_t)i * nn + (wb - n_lo)) * NM & 3);
        __syncthreads();
        wtrace(wt, s, 1);
        // ---- phase 1 (one pass, no barrier inside):
        // (eps, eps) = min(min over the window's nodes c of w(c), lambda1 W^d + alpha_{i+1}(eps, eps)),
        // w(c) = alpha_{i+1}(c, eps) + lambda1 U_i(c): per warp a segmented minimum over the lanes
        // of equal model index (lanes l, l + NM, l + 2 NM, ...), then one atomic per model (w >= 0)
        for (int q0 = warp * 32; q0 < Sw * NM; q0 += KW_THREADS) {
            const int q = q0 + lane;
            float w = INFINITY;
            if (q < Sw * NM) w = msg_n(has_next ? LAY[npp * NM + q] : 0.f, Ui[q]);
            if constexpr (!kMergeDummy)
                if (q < Sw * NM) WC[q] = w;
            for (int o = NM; o < 32; o <<= 1) w = fminf(w, __shfl_down_sync(0xffffffffu, w, o));
            if (lane < NM && q < Sw * NM)
                atomicMin(reinterpret_cast<unsigned *>(DN + 2 * Sw * NM + (q0 + lane) % NM), __float_as_uint(w));
        }
        // messages and every dummy form of row x, one warp per row (measured faster than groups
        // of 4-16 lanes per row on short rows: the per-group redux.sync masks serialise):
        //   m(x, c) = alpha_{i+1}(c, x) + lambda1 U_i(c) + lambda2 Delta -> ENT, with theta(x -> c)
        //   (x, eps) = min(min_c n(x, c), lambda1 W^d + alpha_{i+1}(eps, x))
        //   (eps, x) = min(min_c w(c), lambda1 W^d + alpha_{i+1}(eps, eps)): the row's candidates
        //   c are exactly the nodes of frames (t'x, t'x + T) in the window
        for (int x = warp; x < Sw; x += KW_WARPS) {
            const int c0 = NLO[x], len = NHI[x] - c0, ro = NRO[x], tx = NT[x];
            float mn[NM], wm[NM];
#pragma unroll
            for (int k = 0; k < NM; ++k) mn[k] = wm[k] = INFINITY;
            for (int j = lane; j < len; j += 32) {
                const int c = c0 + j, e = ro + j;
                HGM_DCHECK(c > x && c < Sw && e < npp && NT[c] - tx >= 1 && NT[c] - tx < T);
                const float *dl = DL + (NT[c] - tx) * NM;
                const float *uc = Ui + c * NM;
                if constexpr (kMergeDummy) {
#pragma unroll
                    for (int k = 0; k < NM; ++k)
                        wm[k] = fminf(wm[k], msg_n(has_next ? LAY[(npp + c) * NM + k] : 0.f, uc[k]));
                }
                float ent[EPF];
#pragma unroll
                for (int k = 0; k < NM; ++k) ent[k] = LAY[e * NM + k];  // alpha_{i+1}(c, x)
                if (has_next)
                    msg_build<NM, true>(ent, uc, dl, mn);
                else
                    msg_build<NM, false>(ent, uc, dl, mn);
                ent[NM] = TH[e];
#pragma unroll
                for (int k = NM + 1; k < EPF; ++k) ent[k] = 0.f;
                if constexpr (EPF % 4 == 0) {
#pragma unroll
                    for (int q = 0; q < EPF / 4; ++q)
                        reinterpret_cast<float4 *>(ENT + (size_t)e * EPF)[q] =
                            make_float4(ent[4 * q], ent[4 * q + 1], ent[4 * q + 2], ent[4 * q + 3]);
                } else {
                    *reinterpret_cast<float2 *>(ENT + (size_t)e * EPF) = make_float2(ent[0], ent[1]);
                }
            }
#pragma unroll
            for (int k = 0; k < NM; ++k) {  // n, w >= 0: float order = unsigned bit order
                const float v = __uint_as_float(__reduce_min_sync(0xffffffffu, __float_as_uint(mn[k])));
                float vw = 0.f;
                if constexpr (kMergeDummy) vw = __uint_as_float(__reduce_min_sync(0xffffffffu, __float_as_uint(wm[k])));
                if (lane == k) {
                    const float bean = __fadd_rn(p.l1W, has_next ? LAY[(npp + Sw + x) * NM + k] : 0.f);
                    BEAN[x * NM + k] = bean;                     // the eps candidate of the states (x, a)
                    DN[x * NM + k] = fminf(v, bean);             // (x, eps)
                    if constexpr (kMergeDummy) DN[(Sw + x) * NM + k] = fminf(vw, EEN[k]);  // (eps, x)
                }
            }
        }
        wtrace(wt, s, 6);
        if (tid == 0) bulk_wait_read_all();  // the previous layer's bulk store has read LAY
        wtrace(wt, s, 7);
        __syncthreads();
        wtrace(wt, s, 2);
        if (tid == 0 && s + 1 < nsteps) issue_u(i - 1);  // UR is free: prefetch the next step's row
        // ---- the new dummy forms into LAY (phase 2b reads BEAN, never LAY's dummy slots)
        if constexpr (kMergeDummy) {
            for (int q = tid; q < (2 * Sw + 1) * NM; q += KW_THREADS) LAY[npp * NM + q] = DN[q];
        } else {
            // large batches (NM >= 3): the (eps, x) minima from the per-node w table, one thread per
            // (x, model) scanning the row's candidate nodes, overlapping phase 2b (NM more row
            // reductions per warp made the 50-model context rows slower on short rows)
            for (int q = tid; q < Sw * NM; q += KW_THREADS) {
                const int x = q / NM, k = q - x * NM;
                float r = INFINITY;
                for (int c = NLO[x]; c < NHI[x]; ++c) r = fminf(r, WC[c * NM + k]);  // frames (t'x, t'x + T)
                LAY[(npp + Sw + x) * NM + k] = fminf(r, EEN[k]);
                LAY[(npp + x) * NM + k] = DN[q];  // (x, eps)
            }
            if (tid < NM) LAY[(npp + 2 * Sw) * NM + tid] = DN[2 * Sw * NM + tid];  // (eps, eps)
        }
        wtrace(wt, s, 3);
        // ---- phase 2b: real states, 32-task groups claimed by warps
        // Few tasks for the CTA's threads (small windows): LPT = 2 or 4 lanes share a task, each
        // taking a contiguous share of its candidates, and the shares' minima are combined by
        // shuffles -- min is exact and order-free, so the result is the same bits, while the
        // step's critical path (the longest task) shrinks by LPT.
        const StepConstB kc = *s_kc;
        const int ntask = *s_ntask;
        const int lsh = ntask * 4 <= KW_THREADS ? 2 : (ntask * 2 <= KW_THREADS ? 1 : 0);
        const int LPT = 1 << lsh, sub = lane & (LPT - 1);
        for (;;) {  // (groups dealt round-robin instead of claimed: C1 -0.6 %, context +0.8 %; kept)
            int t0 = 0;
            if (lane == 0) t0 = atomicAdd(s_claim, 32 >> lsh);
            t0 = __shfl_sync(0xffffffffu, t0, 0);
            if (t0 >= ntask) break;
            const int ti = t0 + (lane >> lsh);
            const bool live = ti < ntask;
            const unsigned tk = TASK[live ? ti : ntask - 1];
            const int b = (int)(tk & 0xffffu), a0 = (int)((tk >> 16) & 0x7fffu);
            const bool two = live && (tk >> 31);
            const int a1 = two ? a0 + 1 : a0;
            const int c0 = NLO[b], la = NLO[a0];
            const int trip = live ? NHI[a0] - c0 : 0;
            HGM_DCHECK(!live || (a0 < b && a1 < b && b < Sw && NRO[a1] + (b - la) < npp && NRO[b] + max(trip, 0) <= npp &&
                                 NRO[a0] + (c0 - la) + max(trip, 0) <= npp && NRO[a1] + (c0 - la) + max(trip, 0) <= npp));
            const int aoff = c0 - la, colb = b - la;
            const int ra0 = NRO[a0], ra1 = NRO[a1];
            const float *erow = ENT + (size_t)NRO[b] * EPF;
            const float *arow0 = TH + ra0 + aoff, *arow1 = TH + ra1 + aoff;
            const float th_ab0 = TH[ra0 + colb], th_ab1 = TH[ra1 + colb];
            auto dirty_of = [&](int a) {
                const int lca = NLC[a];
                return lca >= 0 && lca >= min(colb, aoff) && NFC[a] <= max(colb, aoff + trip - 1);
            };
            const bool dirty = live && (dirty_of(a0) || dirty_of(a1) || NFC[b] < trip);
            float R0[NM], R1[NM];
#pragma unroll
            for (int k = 0; k < NM; ++k) R0[k] = R1[k] = INFINITY;
            const int per = (trip + LPT - 1) >> lsh;  // this lane's share [jb, je) of the candidates
            const int jb = min(trip, sub * per), je = min(trip, jb + per);
            if (!__any_sync(0xffffffffu, dirty)) {
                task_loop<NM, EPF>(erow + (size_t)jb * EPF, arow0 + jb, arow1 + jb, th_ab0, th_ab1, je - jb, kc, p.l23,
                                   R0, R1);
            } else {  // exact flag-aware loop (coincident points, R10): NaN directions mark them
                const bool co_ab0 = live && isnan(th_ab0);
                const bool co_ab1 = live && isnan(th_ab1);
                for (int j = jb; j < je; ++j) {
                    float e0[EPF];
                    ld_went<EPF>(erow + (size_t)j * EPF, e0);
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
            for (int o = 1; o < LPT; o <<= 1) {  // combine the shares (lanes of a task are adjacent)
#pragma unroll
                for (int k = 0; k < NM; ++k) {
                    R0[k] = fminf(R0[k], __shfl_xor_sync(0xffffffffu, R0[k], o));
                    R1[k] = fminf(R1[k], __shfl_xor_sync(0xffffffffu, R1[k], o));
                }
            }
            if (live && sub == 0) {
                const int g = NT[b] - NT[a0];
#pragma unroll
                for (int k = 0; k < NM; ++k) {
                    const float sc_g = state_const(p.l2, kc.c[k].y, g);
                    const float ean = BEAN[b * NM + k];
                    LAY[(ra0 + colb) * NM + k] = fminf(__fadd_rn(R0[k], sc_g), ean);
                    if (two) LAY[(ra1 + colb) * NM + k] = fminf(__fadd_rn(R1[k], sc_g), ean);
                }
            }
        }
        wtrace(wt, s, 4);
        fence_async_smem();  // LAY's generic-proxy writes before the bulk store reads them
        __syncthreads();
        wtrace(wt, s, 5);
        if (tid == 0) {  // alpha_i -> the history (layer i - 2), one bulk store
            bulk_s2g(hist + (int64_t)(i - 2) * L + d.off, LAY, lay_bytes);
            bulk_commit();
        }
    }
    if (tid == 0) bulk_wait_all();
}

size_t dp_window_smem(const WinCaps &c, int NM) { return WinPlan(c, NM).total; }

template <int NM, int NT>
static hgm_status launch_w(const SceneView &v, const InstDesc *dinst, int ninst, float *hist, int64_t L, int M,
                           const WinStepPtrs &sp, const float *U, int64_t nn, int64_t n_lo, const DPParams &p,
                           const WinCaps &caps, cudaStream_t s) {
    const size_t smem = dp_window_smem(caps, NM);
    int dev = 0;
    HGM_CUDA(cudaGetDevice(&dev));
    static std::mutex mu;
    static int configured[64];
    {
        std::lock_guard<std::mutex> lk(mu);
        const int d = dev < 0 || dev >= 64 ? 0 : dev;
        if (dev < 0 || dev >= 64 || (int)smem > configured[d]) {
            HGM_CUDA(cudaFuncSetAttribute(k_dp_window<NM, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            if (dev >= 0 && dev < 64) configured[d] = (int)smem;
        }
    }
    static int traced = 0;
    unsigned long long *tbuf = nullptr;
    static const bool trace_env = getenv("HGM_TRACE_W") != nullptr;  // (read once: this runs per launch)
    if (trace_env && !traced) {  // diagnosis: per-step phase times of CTA 0, first launch
        traced = 1;
        cudaMalloc(&tbuf, 256 * 8 * 8);
        cudaMemset(tbuf, 0, 256 * 8 * 8);
        cudaMemcpyToSymbol(g_wtrace, &tbuf, sizeof(tbuf));
    }
    k_dp_window<NM, NT><<<ninst, NT, smem, s>>>(v, dinst, hist, L, M, sp, U, nn, n_lo, p, caps, WinPlan(caps, NM));
    if (tbuf) {
        static unsigned long long h[256 * 8];
        unsigned long long *z = nullptr;
        cudaMemcpy(h, tbuf, sizeof(h), cudaMemcpyDeviceToHost);
        cudaMemcpyToSymbol(g_wtrace, &z, sizeof(z));
        cudaFree(tbuf);
        fprintf(stderr, "HGM_TRACE_W NM %d threads %d windows %d smem %zu; per step (us, thread 0): consts+U, "
                "phase1 (own rows), bulk-store read wait, sync, 2a, 2b, sync\n", NM, NT, ninst, smem);
        for (int st = 0; st < 256 && h[st * 8]; ++st) {
            const unsigned long long *q = h + st * 8;
            fprintf(stderr, "step %3d %7.2f %7.2f %7.2f %7.2f %7.2f %7.2f %7.2f\n", st, (q[1] - q[0]) * 1e-3,
                    (q[6] - q[1]) * 1e-3, (q[7] - q[6]) * 1e-3, (q[2] - q[7]) * 1e-3, (q[3] - q[2]) * 1e-3,
                    (q[4] - q[3]) * 1e-3, (q[5] - q[4]) * 1e-3);
        }
    }
    return HGM_OK;
}

// CTA size: a window's steps are serial, so the warps of an SM are what hides the
// latencies of its phases.  Shared memory bounds the CTAs per SM (k, the window's trellis
// is resident); the CTA size is chosen so that k CTAs bring ~32 warps per SM -- 1024
// threads when one window fills an SM's shared memory (C1: 147 KB) or the launch has fewer
// windows than SMs, 512 at two per SM, else 256.  Register budgets cap it: 1024-thread
// CTAs only for NM <= 2 (64 registers per thread), 512 otherwise.
template <int NM>
static hgm_status launch_nm_w(const SceneView &v, const InstDesc *dinst, int ninst, float *hist, int64_t L, int M,
                              const WinStepPtrs &sp, const float *U, int64_t nn, int64_t n_lo, const DPParams &p,
                              const WinCaps &caps, cudaStream_t s, int nsm, int smem_sm) {
    const size_t smem = dp_window_smem(caps, NM);
    const int per_sm = std::max(1, smem_sm / (int)(smem + 1024));  // CTAs per SM by shared memory
    const int k = ninst < nsm ? 1 : std::min(per_sm, (ninst + nsm - 1) / nsm);
    int nt = k <= 1 ? 1024 : (k == 2 ? 512 : 256);
    if (const char *e = getenv("HGM_WIN_THREADS")) nt = atoi(e);  // tuning knob
    const WinCaps &c = caps;
    if constexpr (NM <= 2) {
        if (nt >= 1024) return launch_w<NM, 1024>(v, dinst, ninst, hist, L, M, sp, U, nn, n_lo, p, c, s);
    }
    if (nt >= 512) return launch_w<NM, 512>(v, dinst, ninst, hist, L, M, sp, U, nn, n_lo, p, c, s);
    return launch_w<NM, 256>(v, dinst, ninst, hist, L, M, sp, U, nn, n_lo, p, c, s);
}

hgm_status launch_dp_window(int NM, const SceneView &v, const InstDesc *dinst, int ninst, float *hist, int64_t L,
                            int M, const WinStepPtrs &sp, const float *U, int64_t nn, int64_t n_lo,
                            const DPParams &p, const WinCaps &caps, cudaStream_t s) {
    if (ninst <= 0 || M < 3) return HGM_OK;
    int dev = 0, nsm = 148, smem_sm = 228 * 1024;
    if (cudaGetDevice(&dev) == cudaSuccess) {
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    }
#define HGM_NMW_CASE(n) \
    case n: return launch_nm_w<n>(v, dinst, ninst, hist, L, M, sp, U, nn, n_lo, p, caps, s, nsm, smem_sm)
    switch (NM) {
        HGM_NMW_CASE(1);
        HGM_NMW_CASE(2);
        HGM_NMW_CASE(3);
        HGM_NMW_CASE(4);
        HGM_NMW_CASE(5);
        HGM_NMW_CASE(6);
        HGM_NMW_CASE(7);
        HGM_NMW_CASE(8);
        default: return fail(HGM_ERR_INVALID_ARGUMENT, "model batch size must be 1..8");
    }
#undef HGM_NMW_CASE
}

}  // namespace hgm
