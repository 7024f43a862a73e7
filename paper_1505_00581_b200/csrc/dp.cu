// dp.cu -- K-DP (recursion step), K-BT (init search + backtrack + appearance
// distance) and K-ARG (per-offset model argmin).
//
// The recursion (Eqs. 10-11), with lambdas explicit:
//   alpha_i(b, a) = min_{c in L(b,a) u {eps}} [ lambda1 U_i(c) + lambda2 D(i; c, b, a)
//                                              + alpha_{i+1}(c, b) ],  alpha_{M+1} = 0
// over the pruned candidate range L(b, a) = [minnode(t'(b)+1), minnode(t'(a)+T))
// (readings R1-R3) and the dummy forms of R5.
//
// State storage per (model, offset) instance and step ("layer"), fp32:
//   [ pair states (b,a) | (b, eps) by b | (eps, a) by a | (eps, eps) ]
// where pair state (b, a) lives at the band index of the pair (a -> b) minus
// the band index of the window's first row.  Every layer of
// every step is kept (alpha history); the argmin beta_i of Eq. 12 is NOT
// stored: K-BT re-evaluates the candidates of the one state it visits per
// step with the same arithmetic (hgm_device.cuh) and takes the first
// candidate equal to the minimum -- exactly the first-strict-minimum rule (R11).
#include <algorithm>
#include <cfloat>
#include <cstdlib>
#include <cstring>

#include "dp_common.cuh"

namespace hgm {

// ------------------------------------------------------------------ K-DP v0
// One thread per state of one instance; candidates streamed from the band.
__global__ void __launch_bounds__(256) k_dp_step(SceneView sc, const InstDesc *__restrict__ inst,
                                                 float *__restrict__ hist, int64_t L, int layer, int has_next,
                                                 StepConst k, const float *__restrict__ U, int64_t n_lo,
                                                 DPParams p) {
    const InstDesc d = inst[blockIdx.y];
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    const int Sw = d.we - d.wb;
    if (s >= d.np + 2 * Sw + 1) return;
    float *cur = hist + (int64_t)layer * L + d.off;
    const float *nxt = has_next ? hist + (int64_t)(layer + 1) * L + d.off : nullptr;
    const float *Ui = U - n_lo;
    float out;
    if (s < d.np) {  // real state (b, a)
        const int p_ba = d.pbase + s;
        const int a = sc.prow[p_ba];
        const int lo_a = sc.first(sc.t[a] + 1);
        const int b = lo_a + (p_ba - sc.qstart[a]);
        const int tb = b < sc.S ? sc.t[b] : 0, ta = sc.t[a];
        if (b >= d.we || tb - ta >= p.T) {
            cur[s] = INFINITY;  // outside this window / beyond this call's T: never read
            return;
        }
        const int c0 = sc.first(tb + 1);
        const int c1 = min(sc.first(ta + p.T), d.we);
        const float th_ab = sc.theta[p_ba];
        const bool co_ab = sc.coinc[p_ba];
        int p_bc = sc.qstart[b];              // pair (b -> c), c = c0 + j
        int p_ac = sc.qstart[a] + (c0 - lo_a); // pair (a -> c)
        float R = INFINITY;
        for (int c = c0; c < c1; ++c, ++p_bc, ++p_ac) {
            const float ncb = msg_n(nxt ? nxt[p_bc - d.pbase] : 0.f, Ui[c]);
            const float m = msg_m(ncb, p.l2, k.g_i, sc.t[c] - tb);
            const bool cbc = sc.coinc[p_bc];
            R = fminf(R, cand_value(m, sc.theta[p_bc], th_ab, sc.theta[p_ac], cbc || co_ab, cbc || sc.coinc[p_ac],
                                   k.A1, k.K2, p.l23));
        }
        const float real = __fadd_rn(R, state_const(p.l2, k.g_im1, tb - ta));
        const float eps = __fadd_rn(p.l1W, nxt ? nxt[d.np + Sw + (b - d.wb)] : 0.f);  // alpha(eps, b)
        out = fminf(real, eps);
    } else if (s < d.np + Sw) {  // (b, eps): D = 0 for every candidate (R5)
        const int b = d.wb + (s - d.np);
        const int tb = sc.t[b];
        const int c0 = sc.first(tb + 1), c1 = min(sc.first(tb + p.T), d.we);
        int p_bc = sc.qstart[b];
        float R = INFINITY;
        for (int c = c0; c < c1; ++c, ++p_bc) R = fminf(R, msg_n(nxt ? nxt[p_bc - d.pbase] : 0.f, Ui[c]));
        out = fminf(R, __fadd_rn(p.l1W, nxt ? nxt[d.np + Sw + (b - d.wb)] : 0.f));
    } else if (s < d.np + 2 * Sw) {  // (eps, a): c constrained by a alone (R5)
        const int a = d.wb + (s - d.np - Sw);
        const int ta = sc.t[a];
        const int c0 = sc.first(ta + 1), c1 = min(sc.first(ta + p.T), d.we);
        float R = INFINITY;
        for (int c = c0; c < c1; ++c) R = fminf(R, msg_n(nxt ? nxt[d.np + (c - d.wb)] : 0.f, Ui[c]));
        out = fminf(R, __fadd_rn(p.l1W, nxt ? nxt[d.np + 2 * Sw] : 0.f));
    } else {  // (eps, eps): unconstrained within the window
        float R = INFINITY;
        for (int c = d.wb; c < d.we; ++c) R = fminf(R, msg_n(nxt ? nxt[d.np + (c - d.wb)] : 0.f, Ui[c]));
        out = fminf(R, __fadd_rn(p.l1W, nxt ? nxt[d.np + 2 * Sw] : 0.f));
    }
    cur[s] = out;
}

// ------------------------------------------------------------------ K-BT v0
// One thread per instance: Eq. 13 init search, Eq. 12 backtrack by
// re-evaluation, appearance distance.
__global__ void k_backtrack(SceneView sc, const InstDesc *__restrict__ inst, int ninst, const float *__restrict__ hist,
                            int64_t L, BTArgs bt, DPParams p) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= ninst) return;
    const InstDesc d = inst[k];
    const int Sw = d.we - d.wb, EPS = -1, M = bt.M;
    auto U = [&](int i, int n) { return bt.U[(int64_t)i * bt.nn + (n - bt.n_lo)]; };     // raw (A)
    auto Us = [&](int i, int n) { return bt.Us[(int64_t)i * bt.nn + (n - bt.n_lo)]; };   // lambda1 U
    auto layer = [&](int i) -> const float * {  // alpha_i for 0-based step i (2..M-1); null = alpha == 0
        return (i >= 2 && i <= M - 1) ? hist + (int64_t)(i - 2) * L + d.off : nullptr;
    };
    auto a_pair = [&](const float *l, int later, int earlier) -> float {
        if (!l) return 0.f;
        const int lo = sc.first(sc.t[earlier] + 1);
        return l[sc.qstart[earlier] + (later - lo) - d.pbase];
    };
    auto a_be = [&](const float *l, int b) { return l ? l[d.np + (b - d.wb)] : 0.f; };
    auto a_ea = [&](const float *l, int a) { return l ? l[d.np + Sw + (a - d.wb)] : 0.f; };
    auto a_ee = [&](const float *l) { return l ? l[d.np + 2 * Sw] : 0.f; };

    // ---- Eq. 13: (z1, z2) = argmin lambda1 U(z1) + lambda1 U(z2) + alpha_3(z2, z1), lexicographic
    int z1b = EPS, z2b = EPS;
    float best = INFINITY;
    if (M == 1) {
        for (int c = d.wb; c <= d.we; ++c) {
            const float v = c < d.we ? Us(0, c) : p.l1W;
            if (v < best) { best = v; z1b = c < d.we ? c : EPS; }
        }
    } else {
        const float *a3 = layer(2);
        for (int z1 = d.wb; z1 <= d.we; ++z1) {
            const bool r1 = z1 < d.we;
            const float u1 = r1 ? Us(0, z1) : p.l1W;
            int c0 = d.wb, c1 = d.we;
            if (r1) {
                c0 = sc.first(sc.t[z1] + 1);
                c1 = min(sc.first(sc.t[z1] + p.T), d.we);
            }
            for (int z2 = c0; z2 <= c1; ++z2) {
                const bool r2 = z2 < c1;
                const float u2 = r2 ? Us(1, z2) : p.l1W;
                float al;
                if (r1 && r2) al = a_pair(a3, z2, z1);
                else if (r1) al = a_ea(a3, z1);
                else if (r2) al = a_be(a3, z2);
                else al = a_ee(a3);
                const float v = __fadd_rn(__fadd_rn(u1, u2), al);
                if (v < best) { best = v; z1b = r1 ? z1 : EPS; z2b = r2 ? z2 : EPS; }
            }
        }
    }
    int64_t *zo = bt.z[0] ? bt.z[0] + (int64_t)d.out * M : nullptr;
    float A = z1b == EPS ? p.W : U(0, z1b);
    if (zo) zo[0] = z1b == EPS ? -1 : sc.id[z1b];
    if (M >= 2) {
        A = __fadd_rn(A, z2b == EPS ? p.W : U(1, z2b));
        if (zo) zo[1] = z2b == EPS ? -1 : sc.id[z2b];
    }
    // ---- Eq. 12: z_i = beta_i(z_{i-1}, z_{i-2}), beta re-evaluated
    int zb = z2b, za = z1b;
    for (int i = 2; i < M; ++i) {
        const float *nx = layer(i + 1);
        const float4 kc = bt.step[0][i];
        int zc = EPS;
        float R = INFINITY;
        if (zb != EPS && za != EPS) {
            const int tb = sc.t[zb], ta = sc.t[za];
            const int lo_a = sc.first(ta + 1);
            const int c0 = sc.first(tb + 1), c1 = min(sc.first(ta + p.T), d.we);
            const int p_ba = sc.qstart[za] + (zb - lo_a);
            const float th_ab = sc.theta[p_ba];
            const bool co_ab = sc.coinc[p_ba];
            int arg = EPS;
            int p_bc = sc.qstart[zb], p_ac = sc.qstart[za] + (c0 - lo_a);
            for (int c = c0; c < c1; ++c, ++p_bc, ++p_ac) {
                const float ncb = msg_n(nx ? nx[p_bc - d.pbase] : 0.f, Us(i, c));
                const float m = msg_m(ncb, p.l2, kc.x, sc.t[c] - tb);
                const bool cbc = sc.coinc[p_bc];
                const float v = cand_value(m, sc.theta[p_bc], th_ab, sc.theta[p_ac], cbc || co_ab,
                                           cbc || sc.coinc[p_ac], kc.z, kc.w, p.l23);
                if (v < R) { R = v; arg = c; }
            }
            const float real = __fadd_rn(R, state_const(p.l2, kc.y, tb - ta));
            const float eps = __fadd_rn(p.l1W, a_ea(nx, zb));
            zc = (real <= eps && arg != EPS) ? arg : EPS;
        } else if (zb != EPS) {
            const int tb = sc.t[zb];
            const int c0 = sc.first(tb + 1), c1 = min(sc.first(tb + p.T), d.we);
            int arg = EPS, p_bc = sc.qstart[zb];
            for (int c = c0; c < c1; ++c, ++p_bc) {
                const float v = msg_n(nx ? nx[p_bc - d.pbase] : 0.f, Us(i, c));
                if (v < R) { R = v; arg = c; }
            }
            zc = (R <= __fadd_rn(p.l1W, a_ea(nx, zb)) && arg != EPS) ? arg : EPS;
        } else {
            int c0 = d.wb, c1 = d.we;
            if (za != EPS) {
                c0 = sc.first(sc.t[za] + 1);
                c1 = min(sc.first(sc.t[za] + p.T), d.we);
            }
            int arg = EPS;
            for (int c = c0; c < c1; ++c) {
                const float v = msg_n(a_be(nx, c), Us(i, c));
                if (v < R) { R = v; arg = c; }
            }
            zc = (R <= __fadd_rn(p.l1W, a_ee(nx)) && arg != EPS) ? arg : EPS;
        }
        A = __fadd_rn(A, zc == EPS ? p.W : U(i, zc));
        if (zo) zo[i] = zc == EPS ? -1 : sc.id[zc];
        za = zb;
        zb = zc;
    }
    if (bt.E[0]) bt.E[0][d.out] = best;
    if (bt.A[0]) bt.A[0][d.out] = A;
}

// ------------------------------------------------------------------ K-ARG
// winner(k) = smallest m attaining min_m score(m, k): min over packed keys
// (float bits << 32 | m); scores are >= 0 so the bit pattern orders like the value.
__global__ void k_offset_argmin(const float *__restrict__ score, int nm, int count, float thr, int32_t *winner,
                                float *best) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= count) return;
    unsigned long long key = ~0ull;
    for (int m = 0; m < nm; ++m) {
        const unsigned long long kk =
            ((unsigned long long)__float_as_uint(score[(int64_t)m * count + k]) << 32) | (unsigned)m;
        key = kk < key ? kk : key;
    }
    const int w = (int)(key & 0xffffffffu);
    const float v = __uint_as_float((unsigned)(key >> 32));
    if (winner) winner[k] = v > thr ? -1 : w;
    if (best) best[k] = v;
}

// Independent chains (f3, "Multiple points 2"): the distance of a model is
// the average of its chains' scores.  S_model[m][k] = mean over chains c of model m
// (chains grouped: chain_first[m] .. chain_first[m+1]) of S_chain[c][k], summed in
// chain order.  One thread per (model, offset).
__global__ void k_chain_mean(const float *__restrict__ S_chain, const int32_t *__restrict__ chain_first,
                             int n_models, int count, float *__restrict__ S_model) {
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= (int64_t)n_models * count) return;
    const int m = (int)(q / count), k = (int)(q % count);
    const int c0 = chain_first[m], c1 = chain_first[m + 1];
    float acc = 0.f;
    for (int c = c0; c < c1; ++c) acc += S_chain[(int64_t)c * count + k];
    S_model[q] = acc / (float)(c1 - c0);
}

hgm_status chain_mean(const float *S_chain, const int32_t *chain_first, int n_models, int count, float *S_model,
                      cudaStream_t s) {
    const int64_t n = (int64_t)n_models * count;
    if (n > 0) k_chain_mean<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(S_chain, chain_first, n_models, count, S_model);
    return HGM_OK;
}

// Recognition vote (f1): block label = label of the block's winning prototype (-1 if
// none); clip label = majority over labelled blocks, ties -> smallest label.  One CTA.
__global__ void __launch_bounds__(256) k_block_vote(const int32_t *__restrict__ winner, int count,
                                                    const int32_t *__restrict__ label, int n_labels,
                                                    int32_t *block_label, int32_t *clip_label) {
    extern __shared__ unsigned hist_[];  // [n_labels]
    for (int q = threadIdx.x; q < n_labels; q += blockDim.x) hist_[q] = 0;
    __syncthreads();
    for (int k = threadIdx.x; k < count; k += blockDim.x) {
        const int w = winner[k];
        const int l = w >= 0 ? label[w] : -1;
        if (block_label) block_label[k] = l;
        if (l >= 0) atomicAdd(&hist_[l], 1u);
    }
    __syncthreads();
    if (threadIdx.x < 32) {  // argmax, ties to the smallest label: key = count << 32 | ~label
        unsigned long long best = 0;
        for (int q = threadIdx.x; q < n_labels; q += 32) {
            const unsigned long long key = ((unsigned long long)hist_[q] << 32) | (0xffffffffu - (unsigned)q);
            if (hist_[q] > 0 && key > best) best = key;
        }
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long y = __shfl_xor_sync(0xffffffffu, best, o);
            if (y > best) best = y;
        }
        if (threadIdx.x == 0 && clip_label) *clip_label = best ? (int)(0xffffffffu - (unsigned)(best & 0xffffffffu)) : -1;
    }
}

hgm_status block_vote(const int32_t *winner, int count, const int32_t *label, int n_labels, int32_t *block_label,
                      int32_t *clip_label, cudaStream_t s) {
    k_block_vote<<<1, 256, sizeof(unsigned) * n_labels, s>>>(winner, count, label, n_labels, block_label, clip_label);
    return HGM_OK;
}

hgm_status offset_argmin(const float *score, int n_models, int count, float threshold, int32_t *winner, float *best,
                         cudaStream_t s) {
    if (count <= 0) return HGM_OK;
    Timer tm(s, K_ARG);
    k_offset_argmin<<<(count + 255) / 256, 256, 0, s>>>(score, n_models, count, threshold, winner, best);
    count_launch(K_ARG);
    HGM_CUDA(cudaGetLastError());
    return HGM_OK;
}
// ------------------------------------------------------------------ v0 launchers
// The v0 kernels (one thread per state / per instance, operands from global
// memory) are kept as an independent second implementation of the same
// arithmetic: tests require K-DP v0 and the batched K-DP to agree bit for bit.
hgm_status launch_dp_v0(const SceneView &v, const InstDesc *dinst, int ninst, int64_t maxNs, float *hist, int64_t L,
                        int layer, bool has_next, const StepConst &kc, const float *U, int64_t n_lo, const DPParams &p,
                        cudaStream_t s) {
    const dim3 grid((unsigned)((maxNs + 255) / 256), (unsigned)ninst);
    k_dp_step<<<grid, 256, 0, s>>>(v, dinst, hist, L, layer, has_next, kc, U, n_lo, p);
    return HGM_OK;
}

hgm_status launch_backtrack_v0(const SceneView &v, const InstDesc *dinst, int ninst, const float *hist, int64_t L,
                               const BTArgs &bt, const DPParams &p, cudaStream_t s) {
    k_backtrack<<<(ninst + 127) / 128, 128, 0, s>>>(v, dinst, ninst, hist, L, bt, p);
    return HGM_OK;
}

}  // namespace hgm
