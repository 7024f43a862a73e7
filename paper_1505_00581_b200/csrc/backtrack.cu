// backtrack.cu -- K-BT: Eq. 13 init search + Eq. 12 backtrack + appearance
// distance, one CTA per window, one warp per model.
//
// The argmin tables beta_i of Eq. 12 are not stored by K-DP.  For the one state
// (z_{i-1}, z_{i-2}) the backtrack visits at step i, the warp re-evaluates the
// state's candidates with the SAME device functions as K-DP (hgm_device.cuh),
// takes the minimum, and picks the first candidate (ascending node index, then
// the dummy) that attains it -- the first-strict-minimum rule of reading R11.
// The arithmetic being identical, the minimum found here is bit-identical to
// the alpha value K-DP stored, so the returned assignment is exactly the one
// the stored beta table would have produced.
#include <algorithm>

#include "dp_common.cuh"

namespace hgm {

struct Best {
    float v;
    int z1, z2;
};
__device__ __forceinline__ bool better(const Best &x, const Best &y) {  // lexicographic (v, z1, z2)
    if (x.v != y.v) return x.v < y.v;
    if (x.z1 != y.z1) return x.z1 < y.z1;
    return x.z2 < y.z2;
}

__device__ __forceinline__ Best shfl_best(const Best &b, int o) {
    return Best{__shfl_xor_sync(0xffffffffu, b.v, o), __shfl_xor_sync(0xffffffffu, b.z1, o),
                __shfl_xor_sync(0xffffffffu, b.z2, o)};
}

// Eq. 13 init search (all models at once) over the slice q = q0, q0 + qs, ... of the
// window's (z1, z2) list -- real pairs are the window's band entries (slot e of the
// alpha_3 layer), then (z1, eps), (eps, z2), (eps, eps) -- each slot's NM values one
// load of the layer's state slot; lexicographic minimum per model over the CTA into
// s_best[k][0] (all threads may read it after the call).
template <int NM>
__device__ __forceinline__ void init_search(const SceneView &sc, const InstDesc &d, const float *__restrict__ hist,
                                            int64_t L, const BTArgs &bt, const DPParams &p, int q0, int qs,
                                            Best (*s_best)[8]) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nthr = blockDim.x;
    const int Sw = d.we - d.wb, M = bt.M, T = p.T, SS = bt.SS;
    const int EPSL = d.we;
    auto Uk = [&](int i, int n, int k) { return __ldg(bt.U + ((int64_t)i * bt.nn + (n - bt.n_lo)) * NM + k); };
    auto Usk = [&](int i, int n, int k) { return __ldg(bt.Us + ((int64_t)i * bt.nn + (n - bt.n_lo)) * NM + k); };
    Best best[NM];
#pragma unroll
    for (int k = 0; k < NM; ++k) best[k] = Best{INFINITY, 0x7fffffff, 0x7fffffff};
    if (M == 1) {
        for (int c = d.wb + q0 + tid; c <= d.we; c += qs) {
#pragma unroll
            for (int k = 0; k < NM; ++k) {
                const Best x{c < d.we ? Usk(0, c, k) : p.l1W, c, 0};
                if (better(x, best[k])) best[k] = x;
            }
        }
    } else {
        const float *a3 = hist + d.off;  // layer i = 2
        const int npp = d.npp;
        for (int q = q0 + tid; q < npp + 2 * Sw + 1; q += qs) {
            int z1 = EPSL, z2 = EPSL, slot;
            bool ok = true;
            if (q < npp) {  // real pair (z1 -> z2): band entry of row z1
                z1 = __ldg(sc.prow_pad + d.ppad + q);
                ok = z1 >= 0;
                if (ok) {
                    const int4 ni = __ldg(sc.ninfo + z1);  // (t', minnode(t'+1), qstart, qpad)
                    z2 = ni.y + (d.ppad + q - ni.w);
                    ok = z2 < d.we && __ldg(sc.t + z2) - ni.x < T;
                }
                slot = q;
            } else if (q < npp + Sw) {  // (z1, eps): alpha_3(eps, z1) is the (eps, a) slot of z1
                z1 = d.wb + (q - npp);
                slot = d.ntail + Sw + (z1 - d.wb);
            } else if (q < npp + 2 * Sw) {  // (eps, z2): alpha_3(z2, eps) is the (b, eps) slot of z2
                z2 = d.wb + (q - npp - Sw);
                slot = d.ntail + (z2 - d.wb);
            } else {
                slot = d.ntail + 2 * Sw;  // (eps, eps)
            }
            if (!ok) continue;
#pragma unroll
            for (int k = 0; k < NM; ++k) {
                const float u1 = z1 < EPSL ? Usk(0, z1, k) : p.l1W;
                const float u2 = z2 < EPSL ? Usk(1, z2, k) : p.l1W;
                const float a = M > 2 ? __ldg(a3 + (int64_t)slot * SS + k) : 0.f;
                const Best x{__fadd_rn(__fadd_rn(u1, u2), a), z1, z2};
                if (better(x, best[k])) best[k] = x;
            }
        }
    }
#pragma unroll
    for (int k = 0; k < NM; ++k) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const Best y = shfl_best(best[k], o);
            if (better(y, best[k])) best[k] = y;
        }
        if (lane == 0) s_best[k][warp] = best[k];
    }
    __syncthreads();
    if (tid < NM) {
        Best b = s_best[tid][0];
        for (int w2 = 1; w2 < (nthr >> 5); ++w2)
            if (better(s_best[tid][w2], b)) b = s_best[tid][w2];
        s_best[tid][0] = b;
    }
    __syncthreads();
}

// Init search split over gridDim.y CTAs per window (dense windows: one CTA would
// serialise hundreds of thousands of pairs); partial minima -> part[(w * P + y) * NM + k].
template <int NM>
__global__ void __launch_bounds__(256) k_bt_init(SceneView sc, const InstDesc *__restrict__ inst,
                                                 const float *__restrict__ hist, int64_t L, BTArgs bt, DPParams p,
                                                 Best *__restrict__ part) {
    __shared__ Best s_best[NM][8];
    const InstDesc d = inst[blockIdx.x];
    init_search<NM>(sc, d, hist, L, bt, p, blockIdx.y * blockDim.x, gridDim.y * blockDim.x, s_best);
    if (threadIdx.x < NM) part[((int64_t)blockIdx.x * gridDim.y + blockIdx.y) * NM + threadIdx.x] = s_best[threadIdx.x][0];
}

// One CTA per window, one warp per model of the batch (blockDim = 32 * max(NM, 4)):
// the init search (here, or its P partial minima from k_bt_init), then the Eq. 12
// backtrack, warp k following model k.
template <int NM>
__global__ void __launch_bounds__(256) k_backtrack(SceneView sc, const InstDesc *__restrict__ inst,
                                                   const float *__restrict__ hist, int64_t L, BTArgs bt,
                                                   DPParams p, const Best *__restrict__ part, int P) {
    __shared__ Best s_best[NM][8];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const InstDesc d = inst[blockIdx.x];
    const int Sw = d.we - d.wb, M = bt.M, T = p.T, SS = bt.SS;
    const int EPSL = d.we;  // dummy label: orders after every real node (R11)
    auto Uk = [&](int i, int n, int k) { return __ldg(bt.U + ((int64_t)i * bt.nn + (n - bt.n_lo)) * NM + k); };
    auto Usk = [&](int i, int n, int k) { return __ldg(bt.Us + ((int64_t)i * bt.nn + (n - bt.n_lo)) * NM + k); };
    auto layer = [&](int i) -> const float * {
        return (i >= 2 && i <= M - 1) ? hist + (int64_t)(i - 2) * L + d.off : nullptr;
    };
    // layer layout (dp_common.cuh): pair state (later, earlier) at qpad[earlier] - ppad + column
    auto atk = [&](const float *l, int s, int k) { return l ? __ldg(l + (int64_t)s * SS + k) : 0.f; };
    if (P == 0) init_search<NM>(sc, d, hist, L, bt, p, 0, blockDim.x, s_best);
    if (warp >= NM) return;
    const int kk = warp;  // this warp's model
    Best bst;
    if (P == 0) {
        bst = s_best[kk][0];
    } else {  // partial minima of k_bt_init; the lexicographic order is total, so any split agrees
        bst = Best{INFINITY, 0x7fffffff, 0x7fffffff};
        for (int y = lane; y < P; y += 32) {
            const Best x = part[((int64_t)blockIdx.x * P + y) * NM + kk];
            if (better(x, bst)) bst = x;
        }
        for (int o = 16; o > 0; o >>= 1) {
            const Best y = shfl_best(bst, o);
            if (better(y, bst)) bst = y;
        }
    }
    auto U = [&](int i, int n) { return Uk(i, n, kk); };     // raw (A)
    auto Us = [&](int i, int n) { return Usk(i, n, kk); };   // lambda1 U (the recursion)
    auto at = [&](const float *l, int s) { return atk(l, s, kk); };
    auto a_be = [&](const float *l, int b) { return at(l, d.ntail + (b - d.wb)); };
    auto a_ea = [&](const float *l, int a) { return at(l, d.ntail + Sw + (a - d.wb)); };
    auto a_ee = [&](const float *l) { return at(l, d.ntail + 2 * Sw); };
    // The backtrack is a chain of M - 2 dependent steps, so its time is the latency of
    // each step's dependent loads.  Per node one int4 (t', minnode(t'+1), qstart, qpad)
    // replaces separate t / first / qstart / qpad loads and is carried from step to step
    // (z_{i-2} <- z_{i-1} <- z_i); the next step's direction theta(z_{i-1} -> z_i), its
    // candidate-range end and z_i's node info are issued together as soon as z_i is known;
    // the padded band's NaN marks coincident pairs (the flags ride on the angles, as in
    // K-DP); the appearance term of z_i is added one step late so its load never stalls
    // the chain (the sum keeps its order i = 0, 1, ..., M-1).
    const int4 NOI = make_int4(0, 0, 0, 0);
    int za = bst.z1, zb = bst.z2;  // z1, z2 (EPSL = dummy)
    int64_t *zo = bt.z[kk] ? bt.z[kk] + (int64_t)d.out * M : nullptr;
    float A = za == EPSL ? p.W : U(0, za);
    if (lane == 0 && zo) zo[0] = za == EPSL ? -1 : sc.id[za];
    float u_pend = 0.f;  // U(i-1, z_{i-1}), added at step i
    if (M >= 2) {
        u_pend = zb == EPSL ? p.W : U(1, zb);
        if (lane == 0 && zo) zo[1] = zb == EPSL ? -1 : sc.id[zb];
    }
    int4 na = za != EPSL ? __ldg(sc.ninfo + za) : NOI, nb = zb != EPSL ? __ldg(sc.ninfo + zb) : NOI;
    // theta(a -> b) (padded band, NaN = coincident) and the candidate-range end of the state
    float th_ab = (za != EPSL && zb != EPSL) ? __ldg(sc.theta_pad + na.w + (zb - na.y)) : 0.f;
    int hi_a = za != EPSL ? sc.first(na.x + T) : 0;
    for (int i = 2; i < M; ++i) {
        const float *nx = layer(i + 1);
        const float4 kc = bt.step[kk][i];
        const bool rb = zb != EPSL, ra = za != EPSL;
        int c0, c1;
        if (rb) {
            c0 = nb.y;
            c1 = min(ra ? hi_a : sc.first(nb.x + T), d.we);
        } else if (ra) {
            c0 = na.y;
            c1 = min(hi_a, d.we);
        } else {
            c0 = d.wb;
            c1 = d.we;
        }
        const bool co_ab = rb && ra && isnan(th_ab);
        const int aoff = ra ? c0 - na.y : 0;
        const int qbp = nb.w - d.ppad, tb = nb.x;
        HGM_DCHECK(c0 >= d.wb && c1 <= d.we && (!rb || c1 <= c0 || (qbp >= 0 && qbp + (c1 - c0) <= d.npp)));
        // the dummy candidate's value does not depend on the real ones: its load goes first
        const float eps_nx = rb ? a_ea(nx, zb) : a_ee(nx);  // alpha_{i+1}(eps, b) or (eps, eps)
        auto value = [&](int c) -> float {
            const int j = c - c0;
            if (rb) {
                const float n = msg_n(at(nx, qbp + j), Us(i, c));
                if (!ra) return n;
                const float m = msg_m(n, p.l2, kc.x, __ldg(sc.t + c) - tb);
                const float th_bc = __ldg(sc.theta_pad + nb.w + j), th_ac = __ldg(sc.theta_pad + na.w + aoff + j);
                const bool cbc = isnan(th_bc);
                return cand_value(m, th_bc, th_ab, th_ac, cbc || co_ab, cbc || isnan(th_ac), kc.z, kc.w, p.l23);
            }
            return msg_n(a_be(nx, c), Us(i, c));
        };
        // minimum and first argmin (ascending c): groups of 4 x 32 candidates, a lane's
        // 4 evaluations independent (their loads overlap); per group the lane keeps its
        // first minimum, the warp the smallest c attaining the group minimum, and a
        // group replaces the running result only if strictly smaller -- the same
        // first argmin as a candidate-by-candidate scan
        float R = INFINITY;
        int arg = -1;
        for (int cb = c0; cb < c1; cb += 128) {
            float v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int c = cb + 32 * u + lane;
                v[u] = c < c1 ? value(c) : INFINITY;
            }
            float lv = v[0];
            int lc = cb + lane;
#pragma unroll
            for (int u = 1; u < 4; ++u)
                if (v[u] < lv) {
                    lv = v[u];
                    lc = cb + 32 * u + lane;
                }
            const float cm = warp_min(lv);
            if (cm < R) {
                R = cm;
                arg = (int)__reduce_min_sync(0xffffffffu, lv == cm ? (unsigned)lc : 0xffffffffu);
            }
        }
        float real = R;
        if (rb && ra) real = __fadd_rn(R, state_const(p.l2, kc.y, tb - na.x));
        const float eps = __fadd_rn(p.l1W, eps_nx);
        const int zc = (arg >= 0 && real <= eps) ? arg : EPSL;
        // next step's operands, all issued at once: node info of z_i, theta(z_{i-1} -> z_i),
        // the candidate-range end of z_{i-1}; U(i, z_i) is summed next step (or after the loop)
        const int4 nc = zc != EPSL ? __ldg(sc.ninfo + zc) : NOI;
        const float th_next = (rb && zc != EPSL) ? __ldg(sc.theta_pad + nb.w + (zc - nb.y)) : 0.f;
        const int hi_next = rb ? sc.first(nb.x + T) : 0;
        A = __fadd_rn(A, u_pend);
        u_pend = zc == EPSL ? p.W : U(i, zc);
        if (lane == 0 && zo) zo[i] = zc == EPSL ? -1 : sc.id[zc];
        za = zb;
        zb = zc;
        na = nb;
        nb = nc;
        th_ab = th_next;
        hi_a = hi_next;
    }
    if (M >= 2) A = __fadd_rn(A, u_pend);
    if (lane == 0) {
        if (bt.E[kk]) bt.E[kk][d.out] = bst.v;
        if (bt.A[kk]) bt.A[kk][d.out] = A;
    }
}

hgm_status launch_backtrack_warp(const SceneView &v, const InstDesc *dinst, int ninst, const float *hist, int64_t L,
                                 const BTArgs &bt, const DPParams &p, cudaStream_t s) {
    if (ninst <= 0) return HGM_OK;
    const int threads = 32 * std::max(bt.NM, 4);  // >= 4 warps for the init search
    // few windows per launch (dense chunks): split their init search over P CTAs each
    const int P = ninst >= 296 ? 0 : std::min(64, (296 + ninst - 1) / ninst);
    DevBuf part;
    if (P > 0) HGM_TRY(part.alloc(sizeof(Best) * (size_t)ninst * P * bt.NM, s));
    Best *pp = P > 0 ? static_cast<Best *>(part.p) : nullptr;
    if (P > 0) count_launch(K_BT);  // the split init search (the caller counts k_backtrack)
#define HGM_BT_CASE(n)                                                                          \
    case n:                                                                                     \
        if (P > 0) k_bt_init<n><<<dim3(ninst, P), 256, 0, s>>>(v, dinst, hist, L, bt, p, pp);     \
        k_backtrack<n><<<ninst, threads, 0, s>>>(v, dinst, hist, L, bt, p, pp, P);              \
        break
    switch (bt.NM) {
        HGM_BT_CASE(1);
        HGM_BT_CASE(2);
        HGM_BT_CASE(3);
        HGM_BT_CASE(4);
        HGM_BT_CASE(5);
        HGM_BT_CASE(6);
        HGM_BT_CASE(7);
        HGM_BT_CASE(8);
        default: return fail(HGM_ERR_INVALID_ARGUMENT, "model batch size must be 1..8");
    }
#undef HGM_BT_CASE
    return HGM_OK;
}

}  // namespace hgm
