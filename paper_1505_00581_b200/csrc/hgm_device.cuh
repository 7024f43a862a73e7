// hgm_device.cuh -- the per-candidate arithmetic of the recursion, shared by the
// DP step kernels (K-DP) and the backtrack (K-BT) so that the backtrack's
// re-evaluation of a minimum is bit-identical to the value the DP stored.
//
// Every operation is an explicit round-to-nearest intrinsic: nvcc may not
// contract, reorder or fast-math any of it, so the same inputs give the same
// bits in every kernel that includes this file.
//
// Method (Eqs. 3-6; DESIGN.md §6 "hoisted form"):
//   For model triple (i, i-1, i-2) and scene triple (c, b, a):
//     D = Delta(i,i-1) + Delta(i-1,i-2) + lambda3 * sqrt(e1^2 + e2^2)
//   e1 = (angle at b)  - (model angle at i-1)
//   e2 = (angle at c)  - (model angle at i)      (sign irrelevant: squared)
//   With theta(u->v) the direction of the ray u->v (atan2f, K-G):
//     angle at b = | |theta(b->c) - theta(a->b)| - pi |          ("fold_b")
//     angle at c = pi - | |theta(b->c) - theta(a->c)| - pi |     (pi - "fold_c")
//   because the unsigned angle between two directions d apart is
//   pi - ||d| - pi| for d in [-2pi, 2pi], and reversing one ray adds pi.
//   A zero-length ray makes the angle 0 (reading R10): fold_b = 0, fold_c = pi.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace hgm {

#define HGM_PI_F 3.14159265358979323846f

__device__ __forceinline__ int first_at(const int32_t *__restrict__ ft, int fmax, int S, int f) {
    // minnode(f): first node with frame >= f, S past the end (R4)
    return f <= 0 ? 0 : (f > fmax ? S : __ldg(ft + f));
}

__device__ __forceinline__ float dir_of(float ax, float ay, float cx, float cy) {
    // direction of the ray a -> c; precise atan2f (not fast-math), atan2f(0,0) = 0
    return atan2f(__fsub_rn(cy, ay), __fsub_rn(cx, ax));
}

__device__ __forceinline__ float fold(float t1, float t2) {
    return fabsf(__fsub_rn(fabsf(__fsub_rn(t1, t2)), HGM_PI_F));
}

// One MUFU.SQRT (the non-.ftz form adds a 3-instruction denormal fix-up; an
// argument below 1.2e-38 contributes < 1.1e-19 to an energy, far below the
// 1e-6 absolute tolerance).
__device__ __forceinline__ float sqrt_approx(float x) {
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// sqrt(e1^2 + e2^2) for the two folds of the scene triple against the
// model constants A1 (model angle at i-1) and K2 (model fold at i).
__device__ __forceinline__ float dg_norm(float fb, float fc, float A1, float K2) {
    float e1 = __fsub_rn(fb, A1);
    float e2 = __fsub_rn(fc, K2);
    return sqrt_approx(__fmaf_rn(e1, e1, __fmul_rn(e2, e2)));
}

// Real-triple candidate value: m(b,c) + lambda2*lambda3 * Dg.
__device__ __forceinline__ float cand_value(float m_bc, float th_bc, float th_ab, float th_ac, bool co_b,
                                            bool co_c, float A1, float K2, float l23) {
    float fb = co_b ? 0.0f : fold(th_bc, th_ab);
    float fc = co_c ? HGM_PI_F : fold(th_bc, th_ac);
    return __fmaf_rn(l23, dg_norm(fb, fc, A1, K2), m_bc);
}

// n(b,c) = alpha_{i+1}(c, b) + lambda1 * U_i(c)   (Eq. 10 without D); l1u_c = lambda1 * U_i(c)
// rounded once by K-U (unary.cu writes the scaled table next to the raw one)
__device__ __forceinline__ float msg_n(float alpha_cb, float l1u_c) { return __fadd_rn(alpha_cb, l1u_c); }

// lambda1 * U, the single rounding every kernel's scaled unary value carries
__device__ __forceinline__ float scale_l1(float l1, float u) { return __fmul_rn(l1, u); }

// lambda2 * Delta(i, i-1) for a frame gap dt = t'(c) - t'(b)
__device__ __forceinline__ float delta_term(float l2, float g_i, int dt_cb) {
    return __fmul_rn(l2, fabsf(__fsub_rn(g_i, (float)dt_cb)));
}

// m(b,c) = n(b,c) + lambda2 * Delta(i, i-1)
__device__ __forceinline__ float msg_m(float n_bc, float l2, float g_i, int dt_cb) {
    return __fadd_rn(n_bc, delta_term(l2, g_i, dt_cb));
}

// lambda2 * Delta(i-1, i-2), added to a real state's minimum after the min
__device__ __forceinline__ float state_const(float l2, float g_im1, int dt_ba) {
    return __fmul_rn(l2, fabsf(__fsub_rn(g_im1, (float)dt_ba)));
}

}  // namespace hgm
