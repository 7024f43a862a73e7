// msg.cu -- K-MSG0: the partial messages of the FIRST recursion step of a chunk.
//
// For step i = M (paper numbering; alpha_{M+1} = 0, Eq. 11) and every real pair
// (x -> c) of the window (c in frames (t'(x), t'(x)+T)):
//   n^k(x, c) = alpha^k_{M+1}(c, x) + lambda1 U^k_M(c) = lambda1 U^k_M(c)
// written into the message buffer in padded band order.  Every later step gets
// its partial messages from the epilogue of the previous K-DP launch
// (dp_batch.cu), with the same msg_n arithmetic.  One warp per window node.
#include <algorithm>

#include "dp_common.cuh"

namespace hgm {

template <int NM>
__global__ void __launch_bounds__(256) k_msg0(SceneView sc, const InstDesc *__restrict__ inst, int T,
                                              const float *__restrict__ Ui, float *__restrict__ msg, float l1) {
    constexpr int NMP = nm_pad(NM);
    const InstDesc d = inst[blockIdx.y];
    const int lane = threadIdx.x & 31;
    const int x = d.wb + blockIdx.x * 8 + (threadIdx.x >> 5);
    if (x >= d.we) return;
    const int tx = sc.t[x];
    const int f1 = sc.first(tx + 1);
    const int len = max(0, min(sc.first(tx + T), d.we) - f1);
    float *row = msg + d.moff + (int64_t)(__ldg(sc.qpad + x) - d.ppad) * NMP;
    for (int j = lane; j < len; j += 32) {
        const int c = f1 + j;
#pragma unroll
        for (int k = 0; k < NM; ++k) row[(int64_t)j * NMP + k] = msg_n(0.f, l1, __ldg(Ui + (int64_t)c * NM + k));
    }
}

hgm_status launch_msg0(int NM, const SceneView &v, const InstDesc *dinst, int ninst, int max_sw, int T,
                       const float *Ui, float *msg, float l1, cudaStream_t s) {
    const dim3 grid((unsigned)std::max(1, (max_sw + 7) / 8), (unsigned)ninst);
#define HGM_NM_CASE(n) \
    case n: k_msg0<n><<<grid, 256, 0, s>>>(v, dinst, T, Ui, msg, l1); break
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
    return HGM_OK;
}

}  // namespace hgm
