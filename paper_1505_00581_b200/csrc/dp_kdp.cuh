// dp_kdp.cuh -- device helpers shared by the K-DP kernels (dp_batch.cu: the batched
// persistent kernel over (window, b-frame tile) items; dp_window.cu: the per-window
// kernel that keeps a window's whole trellis in shared memory for all steps):
// mbarrier / TMA bulk-copy wrappers, candidate-entry loads and the packed (f32x2)
// per-candidate body, which rounds exactly like cand_value() of hgm_device.cuh.
#pragma once
#include "dp_common.cuh"

namespace hgm {

__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~(size_t)15; }

// ------------------------------------------------------------------ TMA bulk copies
__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// try_wait with a short suspend-time hint: the waiting warp sleeps in hardware (no
// polling instructions) and oversleeps the phase completion by at most ~hint_ns (a
// 1 ms hint was seen to oversleep by that much).
// The hint does not keep the warp suspended for long (ncu: the retry loop of the waits was
// ~7 % of K-DP's issued instructions, stealing issue slots from the computing warps), so a
// failed attempt also backs off with __nanosleep before retrying.
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity, unsigned hint_ns = 256,
                                          unsigned backoff_ns = 64) {
    unsigned ok = 0;
    for (;;) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(parity), "r"(hint_ns)
            : "memory");
        if (ok) break;
        __nanosleep(backoff_ns);
    }
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// Bulk copies into one mbarrier's phase: each copy first raises the phase's expected
// transaction count (mbarrier.expect_tx, no arrival), then one arrival closes the
// phase's arrival count once every copy is issued.
struct Copier {
    uint64_t *bar;
    unsigned total = 0;
    __device__ __forceinline__ explicit Copier(uint64_t *b) : bar(b) {}
    __device__ __forceinline__ void raw(void *d, const void *s, unsigned bytes) {
        if (bytes == 0) return;
        asm volatile("mbarrier.expect_tx.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
        bulk_g2s(d, s, bytes, bar);
        total += bytes;
    }
    // Elements [g0, g1) of a 4-byte-element array, widened to whole 16-byte units
    // (the allocations carry >= 16 bytes of slack): dst[q] = src[a0 + q], a0 = g0 & ~3.
    // Returns g0 - a0, the index of element g0 in dst.
    template <class T>
    __device__ __forceinline__ int range(void *d, const T *s, int64_t g0, int64_t g1) {
        static_assert(sizeof(T) == 4, "4-byte elements");
        const int64_t a0 = g0 & ~(int64_t)3, a1 = (g1 + 3) & ~(int64_t)3;
        if (g1 > g0) raw(d, s + a0, (unsigned)((a1 - a0) * 4));
        return (int)(g0 - a0);
    }
    __device__ __forceinline__ void close() {
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
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

// mbarrier helpers beyond the TMA ones
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx_noarrive(uint64_t *bar, unsigned bytes) {
    asm volatile("mbarrier.expect_tx.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

// shared -> global bulk copy (TMA store engine), completion tracked per bulk group of the
// issuing thread; the writes of the source region must be made visible to the async proxy
// first (fence_async_smem by every writing thread, then a CTA barrier)
__device__ __forceinline__ void bulk_s2g(void *gdst, const void *ssrc, unsigned bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(ssrc)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// the source shared memory of every committed bulk store may be overwritten after this
__device__ __forceinline__ void bulk_wait_read_all() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
// every committed bulk store is complete (globally visible to later kernels)
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ void mbar_complete_tx(uint64_t *bar, unsigned n) {
    asm volatile("mbarrier.complete_tx.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(n) : "memory");
}

// Both angle folds of one (candidate, state) in two packed adds: (|t_bc - t_ab| - pi,
// |t_bc - t_ac| - pi) -- subtraction is addition of the negation, so every lane rounds
// exactly like fold() of hgm_device.cuh; the outer |.| becomes an operand modifier of the
// consumer (ptxas: FADD2 R, |R|.F32x2.HI_LO, imm; FADD2 R, |R|.F32, R.F32x2).
__device__ __forceinline__ float2 fold2(float t_bc, float t_ab, float t_ac) {
    const float2 d = __fadd2_rn(make_float2(t_bc, t_bc), make_float2(-t_ab, -t_ac));
    const float2 f = __fadd2_rn(make_float2(fabsf(d.x), fabsf(d.y)), make_float2(-HGM_PI_F, -HGM_PI_F));
    return make_float2(fabsf(f.x), fabsf(f.y));
}

// v_k for candidate entry e (messages e[0..NM), theta(b->c) = e[NM]) of state (b, a)
template <int NM, int E>
__device__ __forceinline__ void cand_entry(const float (&e)[E], float th_ab, float th_ac, const StepConstB &pc,
                                           float l23, float (&v)[NM]) {
    const float2 f = fold2(e[NM], th_ab, th_ac);
    cand_values<NM>(f.x, f.y, e, pc, l23, v);
}

template <int E>
__device__ __forceinline__ void ld_went(const float *__restrict__ src, float (&e)[E]) {
    if constexpr (E % 4 == 0) {
#pragma unroll
        for (int q = 0; q < E / 4; ++q) {
            const float4 v = reinterpret_cast<const float4 *>(src)[q];
            e[4 * q] = v.x;
            e[4 * q + 1] = v.y;
            e[4 * q + 2] = v.z;
            e[4 * q + 3] = v.w;
        }
    } else {
        static_assert(E == 2, "entry of 2 or 4k floats");
        const float2 v = *reinterpret_cast<const float2 *>(src);
        e[0] = v.x;
        e[1] = v.y;
    }
}

// One model, two states (b, a0), (b, a1) of a task against one candidate entry: with a single
// model the two STATES share the packed lanes (the model constants broadcast): folds
// (t_bc - t_ab0, t_bc - t_ab1) and (t_bc - t_ac0, t_bc - t_ac1), then e1, e2, the norm, the
// square roots and the weighted add, each a packed op -- every lane rounds like cand_value().
template <int E>
__device__ __forceinline__ float2 cand_nm1_states(const float (&e)[E], float2 nth_ab, float th_ac0, float th_ac1,
                                                  const StepConstB &pc, float l23) {
    const float tbc = e[1];
    const float2 db = __fadd2_rn(make_float2(tbc, tbc), nth_ab);
    const float2 dc = __fadd2_rn(make_float2(tbc, tbc), make_float2(-th_ac0, -th_ac1));
    const float2 fb = __fadd2_rn(make_float2(fabsf(db.x), fabsf(db.y)), make_float2(-HGM_PI_F, -HGM_PI_F));
    const float2 fc = __fadd2_rn(make_float2(fabsf(dc.x), fabsf(dc.y)), make_float2(-HGM_PI_F, -HGM_PI_F));
    const float2 e1 = __fadd2_rn(make_float2(fabsf(fb.x), fabsf(fb.y)), make_float2(pc.nA1[0].x, pc.nA1[0].x));
    const float2 e2 = __fadd2_rn(make_float2(fabsf(fc.x), fabsf(fc.y)), make_float2(pc.nK2[0].x, pc.nK2[0].x));
    const float2 qq = __ffma2_rn(e1, e1, __fmul2_rn(e2, e2));
    const float2 s = make_float2(sqrt_approx(qq.x), sqrt_approx(qq.y));
    return __ffma2_rn(make_float2(l23, l23), s, make_float2(e[0], e[0]));
}

// The candidate loop of one task (no coincident pair in reach): R0 / R1 = min over the
// trip's candidate entries of the NM model values of states (b, a0) / (b, a1).  Two
// candidates per iteration (3-input mins), entries of E floats (NM messages, theta(b->c)).
template <int NM, int E>
__device__ __forceinline__ void task_loop(const float *__restrict__ erow, const float *__restrict__ arow0,
                                          const float *__restrict__ arow1, float th_ab0, float th_ab1, int trip,
                                          const StepConstB &kc, float l23, float (&R0)[NM], float (&R1)[NM]) {
    int j = 0;
    if constexpr (NM == 1) {
        const float2 nth_ab = make_float2(-th_ab0, -th_ab1);
        for (; j + 1 < trip; j += 2) {
            float e0[E], e1[E];
            ld_went<E>(erow + (size_t)j * E, e0);
            ld_went<E>(erow + (size_t)(j + 1) * E, e1);
            const float2 v0 = cand_nm1_states(e0, nth_ab, arow0[j], arow1[j], kc, l23);
            const float2 v1 = cand_nm1_states(e1, nth_ab, arow0[j + 1], arow1[j + 1], kc, l23);
            R0[0] = min3(R0[0], v0.x, v1.x);
            R1[0] = min3(R1[0], v0.y, v1.y);
        }
        if (j < trip) {
            float e0[E];
            ld_went<E>(erow + (size_t)j * E, e0);
            const float2 v0 = cand_nm1_states(e0, nth_ab, arow0[j], arow1[j], kc, l23);
            R0[0] = fminf(R0[0], v0.x);
            R1[0] = fminf(R1[0], v0.y);
        }
    } else {
        for (; j + 1 < trip; j += 2) {
            float e0[E], e1[E];
            ld_went<E>(erow + (size_t)j * E, e0);
            ld_went<E>(erow + (size_t)(j + 1) * E, e1);
            {
                float v0[NM], v1[NM];
                cand_entry<NM>(e0, th_ab0, arow0[j], kc, l23, v0);
                cand_entry<NM>(e1, th_ab0, arow0[j + 1], kc, l23, v1);
#pragma unroll
                for (int k = 0; k < NM; ++k) R0[k] = min3(R0[k], v0[k], v1[k]);
            }
            {
                float v0[NM], v1[NM];
                cand_entry<NM>(e0, th_ab1, arow1[j], kc, l23, v0);
                cand_entry<NM>(e1, th_ab1, arow1[j + 1], kc, l23, v1);
#pragma unroll
                for (int k = 0; k < NM; ++k) R1[k] = min3(R1[k], v0[k], v1[k]);
            }
        }
        if (j < trip) {
            float e0[E];
            ld_went<E>(erow + (size_t)j * E, e0);
            float v0[NM], v1[NM];
            cand_entry<NM>(e0, th_ab0, arow0[j], kc, l23, v0);
            cand_entry<NM>(e0, th_ab1, arow1[j], kc, l23, v1);
#pragma unroll
            for (int k = 0; k < NM; ++k) {
                R0[k] = fminf(R0[k], v0[k]);
                R1[k] = fminf(R1[k], v1[k]);
            }
        }
    }
}

// Messages of one candidate entry: n_k = alpha_{i+1}(c,b)_k + lambda1 U_i(c)_k (ent[k] holds
// the landed alpha), running minimum of n_k (the (b, eps) state), then m_k = n_k + lambda2
// Delta -- two models per packed add (no multiply left: lambda1 U comes pre-scaled, so no
// FFMA2 contraction can change the rounding); u / dl are 8-byte aligned for even NM.
template <int NM, bool kHasNext>
__device__ __forceinline__ void msg_build(float *ent, const float *__restrict__ u, const float *__restrict__ dl,
                                          float (&mn)[NM]) {
    if constexpr (NM % 2 == 0) {
#pragma unroll
        for (int q = 0; q < NM / 2; ++q) {
            const float2 uu = reinterpret_cast<const float2 *>(u)[q];
            const float2 dd = reinterpret_cast<const float2 *>(dl)[q];
            const float2 n = kHasNext ? __fadd2_rn(make_float2(ent[2 * q], ent[2 * q + 1]), uu) : uu;
            mn[2 * q] = fminf(mn[2 * q], n.x);
            mn[2 * q + 1] = fminf(mn[2 * q + 1], n.y);
            const float2 m = __fadd2_rn(n, dd);
            ent[2 * q] = m.x;
            ent[2 * q + 1] = m.y;
        }
    } else {
#pragma unroll
        for (int k = 0; k < NM; ++k) {
            const float n = kHasNext ? msg_n(ent[k], u[k]) : u[k];
            mn[k] = fminf(mn[k], n);
            ent[k] = __fadd_rn(n, dl[k]);  // msg_m
        }
    }
}

}  // namespace hgm
