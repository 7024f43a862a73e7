// backtrack.cu -- K-BT: Eq. 13 init search + Eq. 12 backtrack + appearance
// distance, one warp per (model, window) pair.
//
// The argmin tables beta_i of Eq. 12 are not stored by K-DP.  For the one state
// (z_{i-1}, z_{i-2}) the backtrack visits at step i, the warp re-evaluates the
// state's candidates with the SAME device functions as K-DP (hgm_device.cuh),
// takes the minimum, and picks the first candidate (ascending node index, then
// the dummy) that attains it -- the first-strict-minimum rule of reading R11.
// The arithmetic being identical, the minimum found here is bit-identical to
// the alpha value K-DP stored, so the returned assignment is exactly the one
// the stored beta table would have produced.
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

__global__ void __launch_bounds__(128) k_backtrack_warp(SceneView sc, const InstDesc *__restrict__ inst, int npairs,
                                                        const float *__restrict__ hist, int64_t L, BTArgs bt,
                                                        DPParams p) {
    const int lane = threadIdx.x & 31;
    const int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (wid >= npairs) return;
    const int NM = bt.NM, kk = wid % NM;
    const InstDesc d = inst[wid / NM];
    const int Sw = d.we - d.wb, M = bt.M, T = p.T;
    const int EPSL = d.we;  // dummy label: orders after every real node (R11)
    auto U = [&](int i, int n) { return __ldg(bt.U + ((int64_t)i * bt.nn + (n - bt.n_lo)) * NM + kk); };
    auto layer = [&](int i) -> const float * {
        return (i >= 2 && i <= M - 1) ? hist + (int64_t)(i - 2) * L + d.off : nullptr;
    };
    auto at = [&](const float *l, int s) { return l ? l[(int64_t)s * bt.SS + kk] : 0.f; };  // state stride SS
    // layer layout (dp_common.cuh): pair state (later, earlier) at qpad[earlier] - ppad + column
    auto a_be = [&](const float *l, int b) { return at(l, d.ntail + (b - d.wb)); };
    auto a_ea = [&](const float *l, int a) { return at(l, d.ntail + Sw + (a - d.wb)); };
    auto a_ee = [&](const float *l) { return at(l, d.ntail + 2 * Sw); };

    // ---- Eq. 13 init search
    Best best{INFINITY, 0x7fffffff, 0x7fffffff};
    if (M == 1) {
        for (int c = d.wb + lane; c <= d.we; c += 32) {
            const Best x{c < d.we ? __fmul_rn(p.l1, U(0, c)) : p.l1W, c, 0};
            if (better(x, best)) best = x;
        }
    } else {
        const float *a3 = layer(2);
        for (int z1 = d.wb + lane; z1 <= d.we; z1 += 32) {
            const bool r1 = z1 < d.we;
            const float u1 = r1 ? __fmul_rn(p.l1, U(0, z1)) : p.l1W;
            int c0 = d.wb, c1 = d.we, q = 0, lo = 0;
            if (r1) {
                lo = sc.first(sc.t[z1] + 1);
                c0 = lo;
                c1 = min(sc.first(sc.t[z1] + T), d.we);
                q = sc.qpad[z1];
            }
            for (int z2 = c0; z2 <= c1; ++z2) {
                const bool r2 = z2 < c1;
                const float u2 = r2 ? __fmul_rn(p.l1, U(1, z2)) : p.l1W;
                float al;
                if (r1 && r2) al = at(a3, q + (z2 - lo) - d.ppad);
                else if (r1) al = a_ea(a3, z1);
                else if (r2) al = a_be(a3, z2);
                else al = a_ee(a3);
                const Best x{__fadd_rn(__fadd_rn(u1, u2), al), z1, r2 ? z2 : EPSL};
                if (better(x, best)) best = x;
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        Best y{__shfl_xor_sync(0xffffffffu, best.v, o), __shfl_xor_sync(0xffffffffu, best.z1, o),
               __shfl_xor_sync(0xffffffffu, best.z2, o)};
        if (better(y, best)) best = y;
    }
    int za = best.z1, zb = best.z2;  // z1, z2 (EPSL = dummy)
    int64_t *zo = bt.z[kk] ? bt.z[kk] + (int64_t)d.out * M : nullptr;
    float A = za == EPSL ? p.W : U(0, za);
    if (lane == 0 && zo) zo[0] = za == EPSL ? -1 : sc.id[za];
    if (M >= 2) {
        A = __fadd_rn(A, zb == EPSL ? p.W : U(1, zb));
        if (lane == 0 && zo) zo[1] = zb == EPSL ? -1 : sc.id[zb];
    }
    // ---- Eq. 12 backtrack, beta_i re-evaluated with the DP's arithmetic
    for (int i = 2; i < M; ++i) {
        const float *nx = layer(i + 1);
        const float4 kc = bt.step[kk][i];
        int c0, c1;
        const bool rb = zb != EPSL, ra = za != EPSL;
        if (rb) {
            c0 = sc.first(sc.t[zb] + 1);
            c1 = min(sc.first((ra ? sc.t[za] : sc.t[zb]) + T), d.we);
        } else if (ra) {
            c0 = sc.first(sc.t[za] + 1);
            c1 = min(sc.first(sc.t[za] + T), d.we);
        } else {
            c0 = d.wb;
            c1 = d.we;
        }
        float th_ab = 0.f;
        bool co_ab = false;
        int qa = 0, qb = 0, qbp = 0, aoff = 0, tb = 0;
        if (rb && ra) {
            qa = sc.qstart[za];
            const int loa = sc.first(sc.t[za] + 1);
            th_ab = sc.theta[qa + (zb - loa)];
            co_ab = sc.coinc[qa + (zb - loa)];
            aoff = c0 - loa;
        }
        if (rb) {
            qb = sc.qstart[zb];
            qbp = sc.qpad[zb] - d.ppad;
            tb = sc.t[zb];
        }
        auto value = [&](int c) -> float {
            const int j = c - c0;
            if (rb) {
                const float n = msg_n(at(nx, qbp + j), p.l1, U(i, c));
                if (!ra) return n;
                const float m = msg_m(n, p.l2, kc.x, sc.t[c] - tb);
                const bool cbc = sc.coinc[qb + j];
                return cand_value(m, sc.theta[qb + j], th_ab, sc.theta[qa + aoff + j], cbc || co_ab,
                                  cbc || sc.coinc[qa + aoff + j], kc.z, kc.w, p.l23);
            }
            return msg_n(a_be(nx, c), p.l1, U(i, c));
        };
        float R = INFINITY;
        for (int c = c0 + lane; c < c1; c += 32) R = fminf(R, value(c));
        R = warp_min(R);
        int arg = -1;
        for (int cb = c0; cb < c1 && arg < 0; cb += 32) {
            const int c = cb + lane;
            const unsigned hit = __ballot_sync(0xffffffffu, c < c1 && value(c) == R);
            if (hit) arg = cb + __ffs(hit) - 1;
        }
        float eps;
        float real = R;
        if (rb && ra) {
            real = __fadd_rn(R, state_const(p.l2, kc.y, tb - sc.t[za]));
            eps = __fadd_rn(p.l1W, a_ea(nx, zb));
        } else if (rb) {
            eps = __fadd_rn(p.l1W, a_ea(nx, zb));
        } else {
            eps = __fadd_rn(p.l1W, a_ee(nx));
        }
        const int zc = (arg >= 0 && real <= eps) ? arg : EPSL;
        A = __fadd_rn(A, zc == EPSL ? p.W : U(i, zc));
        if (lane == 0 && zo) zo[i] = zc == EPSL ? -1 : sc.id[zc];
        za = zb;
        zb = zc;
    }
    if (lane == 0) {
        if (bt.E[kk]) bt.E[kk][d.out] = best.v;
        if (bt.A[kk]) bt.A[kk][d.out] = A;
    }
}

hgm_status launch_backtrack_warp(const SceneView &v, const InstDesc *dinst, int ninst, const float *hist, int64_t L,
                                 const BTArgs &bt, const DPParams &p, cudaStream_t s) {
    const int npairs = ninst * bt.NM;
    k_backtrack_warp<<<(npairs + 3) / 4, 128, 0, s>>>(v, dinst, npairs, hist, L, bt, p);
    return HGM_OK;
}

}  // namespace hgm
