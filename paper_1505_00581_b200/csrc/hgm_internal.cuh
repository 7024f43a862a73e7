// hgm_internal.cuh -- library-internal types of libhgm.so (not part of the ABI).
// Data layout in HBM: DESIGN.md §5.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "../../include/hgm.h"

namespace hgm {

// ------------------------------------------------------------------ errors
void set_error(const std::string &msg);
hgm_status fail(hgm_status st, const std::string &msg);
hgm_status cuda_fail(cudaError_t e, const char *what);

#define HGM_CUDA(call)                                                   \
    do {                                                                 \
        cudaError_t e__ = (call);                                        \
        if (e__ != cudaSuccess) return ::hgm::cuda_fail(e__, #call);     \
    } while (0)

#define HGM_TRY(call)                                                    \
    do {                                                                 \
        hgm_status s__ = (call);                                         \
        if (s__ != HGM_OK) return s__;                                   \
    } while (0)

constexpr int MAX_BATCH_API = 8;
constexpr int HGM_MAX_FRAME = 1 << 26;  // largest accepted frame index (31 days at 25 fps): bounds the frame tables  // models of equal M matched together (dp_common.cuh MAX_BATCH)

// Pad descriptors to a multiple of 4 floats so rows load as float4.
inline int pad4(int F) { return (F + 3) & ~3; }

// RAII device buffer (stream-ordered allocation).
struct DevBuf {
    void *p = nullptr;
    cudaStream_t s = nullptr;
    DevBuf() = default;
    DevBuf(const DevBuf &) = delete;
    DevBuf &operator=(const DevBuf &) = delete;
    ~DevBuf() { release(); }
    hgm_status alloc(size_t bytes, cudaStream_t stream);
    void release();
    template <class T> T *as() const { return static_cast<T *>(p); }
};

}  // namespace hgm

// ------------------------------------------------------------------ handles
// Handle arrays come from the stream-ordered pool.  Every call that reads a
// handle records an event on its stream; hgm_free_* orders the frees after
// those events on a private stream, so releasing a handle never blocks the
// host or idles the GPU (a plain cudaFree synchronises the whole device).
struct HandleUses {
    std::mutex mu;
    std::vector<std::pair<cudaStream_t, cudaEvent_t>> ev;
    void record(cudaStream_t s);
    void release_after(const std::vector<void *> &ptrs, int device);
};

struct hgm_scene {
    mutable HandleUses uses;
    int device = 0;
    int64_t S = 0;     // number of scene nodes
    int F = 0, Fp = 0; // descriptor length, padded length
    int T_max = 1;     // the band covers frame gaps 1..T_max-1
    int fmax = 0;      // last occupied frame; first_tab covers frames [0, fmax+1]
    int64_t npairs = 0;
    // device (sorted by frame, stable)
    int32_t *t = nullptr;
    float *x = nullptr, *y = nullptr;
    float *feat = nullptr;      // [S * Fp]
    int64_t *id = nullptr;      // caller ids of the sorted nodes
    int32_t *first_tab = nullptr; // [fmax + 2]: minnode(f)
    int32_t *qstart = nullptr;  // [S + 1]: start of row a of the pair band
    float *theta = nullptr;     // [npairs]: direction of a -> c (K-G)
    uint8_t *coinc = nullptr;   // [npairs]: 1 if a and c coincide spatially (R10)
    uint16_t *cpre = nullptr;   // [npairs]: inclusive prefix count of coinc along each row
    // padded copy of the band for K-DP staging: row a starts at qpad[a] and has an odd
    // padded length, so consecutive rows fall on distinct shared-memory banks when a
    // tile's rows [A0, B1) are copied as ONE contiguous range
    int32_t *qpad = nullptr;    // [S + 1]
    float *theta_pad = nullptr; // [qpad[S]]
    int32_t *prow_pad = nullptr; // [qpad[S]]: row a of each padded entry, -1 for a padding slot
    int32_t *rfc = nullptr;     // [S]: first coincident column of row a (INT_MAX if none)
    int32_t *rlc = nullptr;     // [S]: last coincident column of row a (-1 if none)
    int4 *ninfo = nullptr;      // [S]: (t'(x), minnode(t'(x)+1), qstart[x], qpad[x]) -- one load per row
    int32_t *prow = nullptr;    // [npairs]: the earlier node a of each pair
    // host mirrors (window / chunk sizing without device round-trips)
    std::vector<int32_t> first_h, qstart_h, qpad_h;
};

struct hgm_model {
    mutable HandleUses uses;
    int device = 0;
    int M = 0, F = 0, Fp = 0;
    int32_t *t = nullptr;
    float *x = nullptr, *y = nullptr;
    float *feat = nullptr;  // [M * Fp]
    float4 *step = nullptr; // [M]: for i >= 2: (g_i, g_{i-1}, A1_i, K2_i), see dp.cu
    std::vector<int32_t> t_h;
    std::vector<float4> step_h;  // host mirror: step constants go into launch parameters
};

namespace hgm {

// ------------------------------------------------------------------ profiling
enum KClass { K_SCENE = 0, K_MODEL = 1, K_UNARY = 2, K_DP = 3, K_BT = 4, K_ARG = 5, K_MSG = 6 };
#include <nvtx3/nvToolsExt.h>

// Host-side enqueue profile (diagnosis, HGM_HOSTPROF=1): wall time the host spends in each
// part of a call, accumulated per slot and printed at process exit (tools/ctx_probe.py).
enum HostSlot { HP_CALL = 0, HP_BATCH, HP_UNARY, HP_PLAN, HP_UPLOAD, HP_DP, HP_BT, HP_LANES, HP_NSLOT };
bool hostprof_on();
void hostprof_add(int slot, double us);
struct HostPhase {
    int slot;
    long long t0;
    explicit HostPhase(int s);
    ~HostPhase();
};

struct NvtxRange {  // host range around an ABI call (no-op unless a tool is attached)
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

struct Timer {  // CUDA events on the launch stream, only when profiling is on; always an NVTX range
    cudaStream_t s;
    int cls;
    cudaEvent_t a = nullptr, b = nullptr;
    Timer(cudaStream_t s_, int cls_);
    ~Timer();
};
void count_launch(int cls, int64_t n = 1);
bool profiling();

// ------------------------------------------------------------------ launchers
hgm_status scene_build_device(const hgm_points *dev_pts, int32_t T_max, cudaStream_t s, hgm_scene **out);
hgm_status model_build_device(const hgm_points *dev_pts, int rank, cudaStream_t s, hgm_model **out);

// Unary table of a batch of NM models of M nodes each (model features stacked
// model-major, node j = k*M + i), batched layout U[((i*nn) + (n - n_lo))*NM + k].
// Us = lambda1 * U (same layout), the recursion's unary term
struct ModelFeats {  // the descriptor tables [M * Fp] of a batch's models (read in place by K-U)
    const float *p[8];
};
hgm_status unary_table(const ModelFeats &mf, int M, int NM, int Fp, const hgm_scene *sc, int64_t n_lo, int64_t n_hi,
                       float l1, float *U, float *Us, cudaStream_t s);
// floats of one table of M x nn x NM (+ 16 B of K-DP bulk-copy slack), 16-byte aligned:
// the raw table at U, the scaled one at U + unary_stride(...)
inline int64_t unary_stride(int M, int NM, int64_t nn) { return ((int64_t)M * NM * nn + 4 + 3) & ~(int64_t)3; }

struct MatchOut {  // per (model, offset) results of one model
    float *E;       // [count] device
    float *A;       // [count] device
    int64_t *z;     // [count * M] device
};
bool use_v0_kernels();
extern thread_local bool g_tiling_failed;  // set by match_batch when a model batch must be split
hgm_status match_batch(const hgm_model *const *models, int NM, const hgm_scene *sc, const hgm_params &pp,
                       const hgm_offsets &o, const float *U, const float *Us, int64_t n_lo, int64_t nn,
                       const MatchOut *outs, cudaStream_t s, int lane = 0);
// lanes of concurrent model batches (detect): lane l > 0 runs on aux_stream(device, l)
// with its own K-DP scratch set
constexpr int MAX_LANES = 8;
cudaStream_t aux_stream(int device, int idx);
hgm_status offset_argmin(const float *score, int n_models, int count, float threshold, int32_t *winner,
                         float *best, cudaStream_t s);
hgm_status chain_mean(const float *S_chain, const int32_t *chain_first, int n_models, int count, float *S_model,
                      cudaStream_t s);
hgm_status block_vote(const int32_t *winner, int count, const int32_t *label, int n_labels, int32_t *block_label,
                      int32_t *clip_label, cudaStream_t s);

}  // namespace hgm
