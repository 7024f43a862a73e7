// api.cu -- the extern "C" surface of libhgm.so (include/hgm.h): argument
// checks, handle ownership, host/device buffer staging, kernel timing.
// All computation happens in the kernels of scene.cu, unary.cu and dp.cu.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <chrono>
#include <memory>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "hgm_internal.cuh"

namespace hgm {

static thread_local std::string g_err;

void set_error(const std::string &msg) { g_err = msg; }
hgm_status fail(hgm_status st, const std::string &msg) {
    g_err = msg;
    return st;
}
hgm_status cuda_fail(cudaError_t e, const char *what) {
    g_err = std::string(what) + ": " + cudaGetErrorString(e);
    cudaGetLastError();  // clear a sticky-free error
    return e == cudaErrorMemoryAllocation ? HGM_ERR_OUT_OF_MEMORY : HGM_ERR_CUDA;
}

hgm_status DevBuf::alloc(size_t bytes, cudaStream_t stream) {
    release();
    s = stream;
    if (bytes == 0) bytes = 16;
    cudaError_t e = cudaMallocAsync(&p, bytes, stream);
    if (e != cudaSuccess) {
        p = nullptr;
        return cuda_fail(e, "cudaMallocAsync");
    }
    return HGM_OK;
}
void DevBuf::release() {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
}

// ------------------------------------------------------------------ profiling
namespace {
std::mutex g_mu;
bool g_prof = false;
struct Pending {
    int cls;
    cudaEvent_t a, b;
};
std::vector<Pending> g_pending;
std::vector<cudaEvent_t> g_event_pool;  // events are reused: creating thousands per step stalls the host
hgm_stats g_stats{};
cudaEvent_t take_event() {  // g_mu held
    if (!g_event_pool.empty()) {
        cudaEvent_t e = g_event_pool.back();
        g_event_pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}
}  // namespace

bool profiling() { return g_prof; }

static const char *const kHostSlot[] = {"detect call", "  per batch (run_batch)", "    unary alloc+launch",
                                         "    match: plan", "    match: uploads", "    match: K-DP launches",
                                         "    match: K-BT launches", "  lanes fork/join"};
static double g_hp_us[HP_NSLOT];
static long long g_hp_n[HP_NSLOT];
static void hostprof_print() {
    fprintf(stderr, "HGM_HOSTPROF host enqueue time per slot (total us, calls, us per call)\n");
    for (int k = 0; k < HP_NSLOT; ++k)
        if (g_hp_n[k])
            fprintf(stderr, "  %-28s %10.1f %8lld %8.2f\n", kHostSlot[k], g_hp_us[k], g_hp_n[k], g_hp_us[k] / g_hp_n[k]);
}
bool hostprof_on() {
    static const bool on = [] {
        const bool e = getenv("HGM_HOSTPROF") && atoi(getenv("HGM_HOSTPROF")) > 0;
        if (e) atexit(hostprof_print);
        return e;
    }();
    return on;
}
static long long now_ns() {
    return std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now().time_since_epoch())
        .count();
}
void hostprof_add(int slot, double us) {
    std::lock_guard<std::mutex> lk(g_mu);
    g_hp_us[slot] += us;
    g_hp_n[slot] += 1;
}
HostPhase::HostPhase(int s) : slot(s), t0(hostprof_on() ? now_ns() : 0) {}
HostPhase::~HostPhase() {
    if (t0) hostprof_add(slot, (now_ns() - t0) * 1e-3);
}

// NVTX ranges (SURVEY.md §5 tracing): every phase timer also opens a host range named after
// its kernel class, so an nsys / ncu --nvtx timeline shows the scene build, unary table,
// recursion, backtrack and argmin of each call; NVTX3 is header-only and its calls are
// no-ops unless a tool is attached.
static const char *const kPhaseName[] = {"hgm:scene (K-G)", "hgm:model", "hgm:unary (K-U)", "hgm:recursion (K-DP)",
                                         "hgm:backtrack (K-BT)", "hgm:argmin (K-ARG)", "hgm:messages"};
Timer::Timer(cudaStream_t s_, int cls_) : s(s_), cls(cls_) {
    nvtxRangePushA(kPhaseName[cls_ >= 0 && cls_ <= K_MSG ? cls_ : 0]);
    if (!g_prof) return;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        a = take_event();
        b = take_event();
    }
    cudaEventRecord(a, s);
}
Timer::~Timer() {
    nvtxRangePop();
    if (!a) return;
    cudaEventRecord(b, s);
    std::lock_guard<std::mutex> lk(g_mu);
    g_pending.push_back({cls, a, b});
}

void count_launch(int cls, int64_t n) {
    std::lock_guard<std::mutex> lk(g_mu);
    g_stats.launches[cls] += n;
    if (cls == K_DP) g_stats.dp_launches += n;
}

}  // namespace hgm

// ------------------------------------------------------------------ handle lifetime
static cudaStream_t free_stream(int device) {
    static std::mutex mu;
    static cudaStream_t fs[64] = {};
    std::lock_guard<std::mutex> lk(mu);
    if (device < 0 || device >= 64) return nullptr;
    if (!fs[device]) cudaStreamCreateWithFlags(&fs[device], cudaStreamNonBlocking);
    return fs[device];
}

void HandleUses::record(cudaStream_t s) {
    std::lock_guard<std::mutex> lk(mu);
    for (auto &pr : ev)
        if (pr.first == s) {
            cudaEventRecord(pr.second, s);
            return;
        }
    cudaEvent_t e;
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return;
    cudaEventRecord(e, s);
    ev.emplace_back(s, e);
}

void HandleUses::release_after(const std::vector<void *> &ptrs, int device) {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    cudaStream_t fs = free_stream(device);
    {
        std::lock_guard<std::mutex> lk(mu);
        for (auto &pr : ev) {
            cudaStreamWaitEvent(fs, pr.second, 0);  // after every call that used the handle
            cudaEventDestroy(pr.second);
        }
        ev.clear();
    }
    for (void *p : ptrs)
        if (p) cudaFreeAsync(p, fs);
    cudaGetLastError();
    cudaSetDevice(prev);
}

using namespace hgm;

// ------------------------------------------------------------------ helpers
static bool is_device_ptr(const void *p) {
    if (!p) return false;
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

static hgm_status check_points(const hgm_points *pts) {
    if (!pts) return fail(HGM_ERR_INVALID_ARGUMENT, "points == NULL");
    if (pts->n <= 0) return fail(HGM_ERR_EMPTY_POINT_SET, "empty point set");
    if (pts->F < 1) return fail(HGM_ERR_INVALID_ARGUMENT, "descriptor length F < 1");
    if (!pts->frame || !pts->x || !pts->y || !pts->feat) return fail(HGM_ERR_INVALID_ARGUMENT, "NULL point array");
    return HGM_OK;
}

static hgm_status check_params(const hgm_params *p, const hgm_scene *sc) {
    if (!p) return fail(HGM_ERR_INVALID_ARGUMENT, "params == NULL");
    const float v[4] = {p->lambda1, p->lambda2, p->lambda3, p->w_dummy};
    for (float x : v)
        if (!std::isfinite(x) || x < 0.f) return fail(HGM_ERR_INVALID_ARGUMENT, "lambda / W^d must be finite and >= 0");
    if (p->T < 1) return fail(HGM_ERR_INVALID_ARGUMENT, "T < 1");
    if (sc && p->T > sc->T_max) return fail(HGM_ERR_INVALID_ARGUMENT, "T exceeds the scene index T_max");
    return HGM_OK;
}

static hgm_status check_offsets(const hgm_offsets *o) {
    if (!o) return fail(HGM_ERR_INVALID_ARGUMENT, "offsets == NULL");
    if (o->window < 1 || o->stride < 1 || o->count < 0)
        return fail(HGM_ERR_INVALID_ARGUMENT, "window < 1, stride < 1 or count < 0");
    // every window frame (and frame + T inside the kernels) must stay far inside int32
    const int64_t last = (int64_t)o->first_frame + (int64_t)(o->count > 0 ? o->count - 1 : 0) * o->stride + o->window;
    if ((int64_t)o->first_frame < -(int64_t)HGM_MAX_FRAME || last > 2 * (int64_t)HGM_MAX_FRAME)
        return fail(HGM_ERR_INVALID_ARGUMENT, "offsets reach beyond +-2^26 frames");
    return HGM_OK;
}

// T at or above the scene's frame span + 1 admits every pair (t'(c) - t'(a) <= fmax < T):
// the kernels run with min(T, fmax + 1), the same result without int overflow in t + T
static hgm_params effective_params(const hgm_params *p, const hgm_scene *sc) {
    hgm_params e = *p;
    e.T = (int32_t)std::min<int64_t>(e.T, (int64_t)sc->fmax + 1);
    return e;
}

// Copy a host point set to the device (borrowed input, copied per the ABI).
struct DevPoints {
    DevBuf frame, x, y, sal, feat, id;
    hgm_points v{};
    hgm_status load(const hgm_points *h, cudaStream_t s) {
        const int64_t n = h->n;
        HGM_TRY(frame.alloc(sizeof(int32_t) * n, s));
        HGM_TRY(x.alloc(sizeof(float) * n, s));
        HGM_TRY(y.alloc(sizeof(float) * n, s));
        HGM_TRY(sal.alloc(sizeof(float) * n, s));
        HGM_TRY(feat.alloc(sizeof(float) * n * h->F, s));
        HGM_CUDA(cudaMemcpyAsync(frame.p, h->frame, sizeof(int32_t) * n, cudaMemcpyHostToDevice, s));
        HGM_CUDA(cudaMemcpyAsync(x.p, h->x, sizeof(float) * n, cudaMemcpyHostToDevice, s));
        HGM_CUDA(cudaMemcpyAsync(y.p, h->y, sizeof(float) * n, cudaMemcpyHostToDevice, s));
        if (h->saliency) {
            HGM_CUDA(cudaMemcpyAsync(sal.p, h->saliency, sizeof(float) * n, cudaMemcpyHostToDevice, s));
        } else {
            HGM_CUDA(cudaMemsetAsync(sal.p, 0, sizeof(float) * n, s));
        }
        HGM_CUDA(cudaMemcpyAsync(feat.p, h->feat, sizeof(float) * n * h->F, cudaMemcpyHostToDevice, s));
        v = *h;
        v.frame = frame.as<int32_t>();
        v.x = x.as<float>();
        v.y = y.as<float>();
        v.saliency = sal.as<float>();
        v.feat = feat.as<float>();
        v.id = nullptr;
        if (h->id) {
            HGM_TRY(id.alloc(sizeof(int64_t) * n, s));
            HGM_CUDA(cudaMemcpyAsync(id.p, h->id, sizeof(int64_t) * n, cudaMemcpyHostToDevice, s));
            v.id = id.as<int64_t>();
        }
        return HGM_OK;
    }
};

// A persistent private stream per device for the synchronous host-input builders
// (creating and destroying a stream per call stalled the host now and then).
static cudaStream_t builder_stream(int device) {
    static std::mutex mu;
    static cudaStream_t bs[64] = {};
    std::lock_guard<std::mutex> lk(mu);
    const int d = device < 0 || device >= 64 ? 0 : device;
    if (!bs[d]) cudaStreamCreateWithFlags(&bs[d], cudaStreamNonBlocking);
    return bs[d];
}
struct StreamGuard {
    cudaStream_t s = nullptr;
};

// Keep freed stream-ordered allocations in the device pool (no release to the
// OS at synchronisation points): the per-call scratch (unary table, alpha
// history, up to a few GB) is then recycled instead of re-mapped every call.
static void configure_pool() {
    static std::mutex mu;
    static bool done[64] = {false};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return;
    std::lock_guard<std::mutex> lk(mu);
    if (done[dev]) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        // Pre-map 4 GiB into the pool once: later per-call allocations (point copies, scene
        // arrays, unary tables) are carved from memory that is already mapped instead of
        // mapping fresh pages mid-call (seen as 100-1000 ms host stalls).
        cudaStream_t st = nullptr;
        if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) == cudaSuccess) {
            void *p = nullptr;
            if (cudaMallocAsync(&p, (size_t)4 << 30, st) == cudaSuccess) cudaFreeAsync(p, st);
            cudaStreamSynchronize(st);
            cudaStreamDestroy(st);
        }
    }
    cudaGetLastError();
    done[dev] = true;
}

static inline int host_first(const hgm_scene *sc, int64_t f) {
    if (f <= 0) return 0;
    if (f > sc->fmax) return (int)sc->S;
    return sc->first_h[f];
}

// ------------------------------------------------------------------ ABI
extern "C" {

const char *hgm_last_error(void) { return g_err.c_str(); }
const char *hgm_version(void) { return "hgm 0.1 (sm_100a)"; }

hgm_status hgm_build_model_graph(const hgm_points *pts, int device, hgm_model **out) {
    NvtxRange nvtx_("hgm_build_model_graph");
    HGM_TRY(check_points(pts));
    if (!out) return fail(HGM_ERR_INVALID_ARGUMENT, "out == NULL");
    HGM_CUDA(cudaSetDevice(device));
    configure_pool();
    StreamGuard sg;
    sg.s = builder_stream(device);
    hgm_status st;
    {
        DevPoints dp;
        HGM_TRY(dp.load(pts, sg.s));
        st = model_build_device(&dp.v, 0, sg.s, out);
    }
    HGM_CUDA(cudaStreamSynchronize(sg.s));
    return st;
}

hgm_status hgm_build_model_graph_dev(const hgm_points *pts, void *stream, hgm_model **out) {
    HGM_TRY(check_points(pts));
    if (!out) return fail(HGM_ERR_INVALID_ARGUMENT, "out == NULL");
    configure_pool();
    return model_build_device(pts, 0, (cudaStream_t)stream, out);
}

hgm_status hgm_build_model_chain(const hgm_points *pts, int device, int32_t rank, hgm_model **out) {
    NvtxRange nvtx_("hgm_build_model_chain");
    HGM_TRY(check_points(pts));
    if (!out) return fail(HGM_ERR_INVALID_ARGUMENT, "out == NULL");
    if (rank < 0) return fail(HGM_ERR_INVALID_ARGUMENT, "rank < 0");
    HGM_CUDA(cudaSetDevice(device));
    configure_pool();
    StreamGuard sg;
    sg.s = builder_stream(device);
    hgm_status st;
    {
        DevPoints dp;
        HGM_TRY(dp.load(pts, sg.s));
        st = model_build_device(&dp.v, rank, sg.s, out);
    }
    HGM_CUDA(cudaStreamSynchronize(sg.s));
    return st;
}

hgm_status hgm_model_num_nodes(const hgm_model *m, int32_t *M) {
    if (!m || !M) return fail(HGM_ERR_INVALID_ARGUMENT, "NULL argument");
    *M = m->M;
    return HGM_OK;
}

void hgm_free_model(hgm_model *m) {
    if (!m) return;
    m->uses.release_after({m->t, m->x, m->y, m->feat, m->step}, m->device);
    delete m;
}

hgm_status hgm_build_scene_index(const hgm_points *pts, int device, int32_t T_max, hgm_scene **out) {
    NvtxRange nvtx_("hgm_build_scene_index");
    HGM_TRY(check_points(pts));
    if (!out) return fail(HGM_ERR_INVALID_ARGUMENT, "out == NULL");
    if (T_max < 1) return fail(HGM_ERR_INVALID_ARGUMENT, "T_max < 1");
    HGM_CUDA(cudaSetDevice(device));
    configure_pool();
    StreamGuard sg;
    sg.s = builder_stream(device);
    hgm_status st;
    {
        DevPoints dp;
        HGM_TRY(dp.load(pts, sg.s));
        st = scene_build_device(&dp.v, T_max, sg.s, out);
    }
    HGM_CUDA(cudaStreamSynchronize(sg.s));
    return st;
}

hgm_status hgm_build_scene_index_dev(const hgm_points *pts, int32_t T_max, void *stream, hgm_scene **out) {
    HGM_TRY(check_points(pts));
    if (!out) return fail(HGM_ERR_INVALID_ARGUMENT, "out == NULL");
    if (T_max < 1) return fail(HGM_ERR_INVALID_ARGUMENT, "T_max < 1");
    configure_pool();
    return scene_build_device(pts, T_max, (cudaStream_t)stream, out);
}

hgm_status hgm_scene_num_nodes(const hgm_scene *sc, int64_t *S) {
    if (!sc || !S) return fail(HGM_ERR_INVALID_ARGUMENT, "NULL argument");
    *S = sc->S;
    return HGM_OK;
}

void hgm_free_scene(hgm_scene *sc) {
    if (!sc) return;
    sc->uses.release_after({sc->t, sc->x, sc->y, sc->feat, sc->id, sc->first_tab, sc->qstart, sc->theta, sc->coinc,
                            sc->cpre, sc->prow, sc->qpad, sc->theta_pad, sc->prow_pad, sc->rfc, sc->rlc,
                            sc->ninfo},
                           sc->device);
    delete sc;
}

// node range covered by all windows of `o`
static void covered_range(const hgm_scene *sc, const hgm_offsets *o, int64_t *lo, int64_t *hi) {
    const int64_t last = (int64_t)o->first_frame + (int64_t)(o->count - 1) * o->stride;
    *lo = host_first(sc, o->first_frame);
    *hi = host_first(sc, last + o->window);
}

hgm_status hgm_match_model_at_offsets(const hgm_model *model, const hgm_scene *scene, const hgm_params *params,
                                      const hgm_offsets *offsets, float *E, float *A, int64_t *z, void *stream) {
    NvtxRange nvtx_("hgm_match_model_at_offsets");
    if (!model || !scene) return fail(HGM_ERR_INVALID_ARGUMENT, "NULL handle");
    HGM_TRY(check_params(params, scene));
    HGM_TRY(check_offsets(offsets));
    if (model->F != scene->F) return fail(HGM_ERR_DIMENSION_MISMATCH, "model and scene descriptor lengths differ");
    const int count = offsets->count;
    if (count == 0) return HGM_OK;
    cudaStream_t s = (cudaStream_t)stream;
    HGM_CUDA(cudaSetDevice(scene->device));
    configure_pool();
    int64_t n_lo, n_hi;
    covered_range(scene, offsets, &n_lo, &n_hi);
    const int64_t nn = std::max<int64_t>(n_hi - n_lo, 1);
    DevBuf U, dE, dA, dz;
    const int64_t ustr = unary_stride(model->M, 1, nn);  // raw U, then lambda1 U
    HGM_TRY(U.alloc(sizeof(float) * 2 * (size_t)ustr, s));
    ModelFeats mf1{};
    mf1.p[0] = model->feat;
    HGM_TRY(unary_table(mf1, model->M, 1, model->Fp, scene, n_lo, n_hi, params->lambda1, U.as<float>(),
                        U.as<float>() + ustr, s));
    const bool hE = E && !is_device_ptr(E), hA = A && !is_device_ptr(A), hz = z && !is_device_ptr(z);
    if (hE) HGM_TRY(dE.alloc(sizeof(float) * count, s));
    if (hA) HGM_TRY(dA.alloc(sizeof(float) * count, s));
    if (hz) HGM_TRY(dz.alloc(sizeof(int64_t) * (size_t)count * model->M, s));
    MatchOut mo{hE ? dE.as<float>() : E, hA ? dA.as<float>() : A, hz ? dz.as<int64_t>() : z};
    const hgm_params pe = effective_params(params, scene);
    HGM_TRY(match_batch(&model, 1, scene, pe, *offsets, U.as<float>(), U.as<float>() + ustr, n_lo, nn, &mo, s));
    scene->uses.record(s);
    model->uses.record(s);
    if (hE) HGM_CUDA(cudaMemcpyAsync(E, dE.p, sizeof(float) * count, cudaMemcpyDeviceToHost, s));
    if (hA) HGM_CUDA(cudaMemcpyAsync(A, dA.p, sizeof(float) * count, cudaMemcpyDeviceToHost, s));
    if (hz) HGM_CUDA(cudaMemcpyAsync(z, dz.p, sizeof(int64_t) * count * model->M, cudaMemcpyDeviceToHost, s));
    if (hE || hA || hz) HGM_CUDA(cudaStreamSynchronize(s));
    HGM_CUDA(cudaGetLastError());
    return HGM_OK;
}

// One model batch [m0, m1) of equal chain length on stream s (lane: its K-DP scratch set),
// E* / A into Ed / Ad [n_models][count], assignments into the scratch zb.  A batch too
// dense for a shared stage (g_tiling_failed) is retried one model at a time.
// floats of a batch's unary region (raw + scaled tables), enough for the batch or for its
// models one at a time (the dense-frame retry below)
static int64_t unary_region(int M, int NM, int64_t nn) { return (2 * ((int64_t)M * NM * nn + 8 * NM) + 3) & ~(int64_t)3; }

static hgm_status run_batch(const hgm_model *const *models, int m0, int m1, const hgm_scene *scene,
                            const hgm_params *params, const hgm_offsets *offsets, int64_t n_lo, int64_t n_hi,
                            float *Ed, float *Ad, int64_t *zb, int Mmax, cudaStream_t s, int lane, float *ureg) {
    HostPhase hp_batch(HP_BATCH);
    const int count = offsets->count, Fp = scene->Fp;
    const int64_t nn = std::max<int64_t>(n_hi - n_lo, 1);
    const hgm_params pe = effective_params(params, scene);
    int max_batch = m1 - m0;
    int64_t uoff = 0;  // next table in the batch's preallocated unary region (detect_scores)
    for (int a = m0; a < m1;) {
        const int b = std::min(m1, a + max_batch);
        const int NM = b - a, M = models[a]->M;
        std::unique_ptr<HostPhase> hp_u(new HostPhase(HP_UNARY));
        ModelFeats mf{};  // K-U reads each model's descriptors in place (no gather copies per batch)
        for (int k = 0; k < NM; ++k) mf.p[k] = models[a + k]->feat;
        const int64_t ustr = unary_stride(M, NM, nn);  // raw U, then lambda1 U
        float *const Ut = ureg + uoff;  // raw U at Ut, lambda1 U at Ut + ustr
        uoff += 2 * ustr;
        HGM_TRY(unary_table(mf, M, NM, Fp, scene, n_lo, n_hi, params->lambda1, Ut,
                            Ut + ustr, s));
        hp_u.reset();
        MatchOut mo[MAX_BATCH_API];
        for (int k = 0; k < NM; ++k)
            mo[k] = MatchOut{Ed + (size_t)(a + k) * count, Ad + (size_t)(a + k) * count, zb + (size_t)k * count * Mmax};
        g_tiling_failed = false;
        const hgm_status bst =
            match_batch(models + a, NM, scene, pe, *offsets, Ut, Ut + ustr, n_lo, nn, mo, s, lane);
        if (bst != HGM_OK && g_tiling_failed && NM > 1) {
            if (getenv("HGM_DEBUG_TILING")) fprintf(stderr, "tiling: batch of %d retried one model at a time\n", NM);
            max_batch = 1;  // too dense for a batch's stage: one model at a time from here on
            uoff = 0;       // (stream order: the retry's tables overwrite the failed batch's)
            continue;
        }
        HGM_TRY(bst);
        a = b;
    }
    return HGM_OK;
}

// Host worker pool for the concurrent model batches of a detect call: each lane's enqueue
// (allocations, planning, ~10 CUDA runtime calls per batch, ~50 us of host time: HGM_HOSTPROF)
// runs on its own host thread, so a call with 7 batches enqueues in about one batch's time.
// Workers are created once and park on a condition variable; lane 0 runs on the caller.  A
// call that finds the pool busy (another host thread's detect) enqueues its lanes serially.
class LanePool {
  public:
    ~LanePool() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto &t : th_) t.join();
    }
    // fn(0) on the calling thread, fn(1..n-1) on workers; returns when all are done
    void run(int n, const std::function<void(int)> &fn) {
        std::unique_lock<std::mutex> busy(run_mu_, std::try_to_lock);
        if (!busy.owns_lock() || n <= 1) {
            for (int l = 0; l < n; ++l) fn(l);
            return;
        }
        {
            std::lock_guard<std::mutex> lk(mu_);
            while ((int)th_.size() < n - 1) th_.emplace_back([this] { work(); });
            job_ = &fn;
            next_ = 1;
            njob_ = n;
            pending_ = n - 1;
            ++gen_;
        }
        cv_.notify_all();
        fn(0);
        std::unique_lock<std::mutex> lk(mu_);
        done_.wait(lk, [this] { return pending_ == 0; });
        job_ = nullptr;
    }

  private:
    void work() {
        uint64_t seen = 0;
        std::unique_lock<std::mutex> lk(mu_);
        for (;;) {
            cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
            if (stop_) return;
            seen = gen_;
            while (job_ && next_ < njob_) {
                const int l = next_++;
                const std::function<void(int)> *fn = job_;
                lk.unlock();
                (*fn)(l);
                lk.lock();
                if (--pending_ == 0) done_.notify_all();
            }
        }
    }
    std::mutex run_mu_, mu_;
    std::condition_variable cv_, done_;
    std::vector<std::thread> th_;
    const std::function<void(int)> *job_ = nullptr;
    int next_ = 0, njob_ = 0, pending_ = 0;
    uint64_t gen_ = 0;
    bool stop_ = false;
};
static LanePool &lane_pool() {
    static LanePool *p = new LanePool();  // never destroyed: workers may outlive static teardown order
    return *p;
}

// E* and A of every (model, offset) into device matrices Ed / Ad [n_models][count].
// Consecutive models of equal chain length form batches of up to MAX_BATCH_API (one K-DP
// pass each).  When the call has few windows (count < 2 x SMs: one batch cannot fill the
// GPU -- the paper's context of 50 models against 60-frame blocks, streaming pushes) the
// batches run CONCURRENTLY, one lane (stream + scratch set) each, forked from and joined
// back into the caller's stream; otherwise one after another on it.
static hgm_status detect_scores(const hgm_model *const *models, int32_t n_models, const hgm_scene *scene,
                                const hgm_params *params, const hgm_offsets *offsets, float *Ed, float *Ad,
                                cudaStream_t s) {
    HostPhase hp_call(HP_CALL);
    const int count = offsets->count;
    configure_pool();
    int64_t n_lo, n_hi;
    covered_range(scene, offsets, &n_lo, &n_hi);
    int Mmax = 0;
    for (int m = 0; m < n_models; ++m) Mmax = std::max(Mmax, models[m]->M);
    const int max_batch = use_v0_kernels() ? 1 : MAX_BATCH_API;
    std::vector<std::pair<int, int>> batches;
    for (int m0 = 0; m0 < n_models;) {
        int m1 = m0 + 1;
        while (m1 < n_models && m1 - m0 < max_batch && models[m1]->M == models[m0]->M) ++m1;
        batches.emplace_back(m0, m1);
        m0 = m1;
    }
    const int nb = (int)batches.size();
    int nsm = 148;
    HGM_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, scene->device));
    const char *lenv = getenv("HGM_LANES");  // 1: batches one after another (tuning / tests)
    int nlane = (nb > 1 && !use_v0_kernels() && count < 2 * nsm) ? std::min(nb, MAX_LANES) : 1;
    if (lenv && atoi(lenv) >= 1) nlane = std::min({nb, MAX_LANES, atoi(lenv)});
    DevBuf zb, Uall;  // one allocation for every batch's unary tables (an allocation per batch
                      // was ~20 us of host time each, and contended between the lanes' threads)
    const size_t zlane = (size_t)count * Mmax * MAX_BATCH_API;
    HGM_TRY(zb.alloc(sizeof(int64_t) * zlane * nlane, s));
    const int64_t nn = std::max<int64_t>(n_hi - n_lo, 1);
    std::vector<int64_t> uofs((size_t)nb + 1, 0);
    for (int bi = 0; bi < nb; ++bi)
        uofs[(size_t)bi + 1] = uofs[(size_t)bi] + unary_region(models[batches[bi].first]->M,
                                                               batches[bi].second - batches[bi].first, nn);
    HGM_TRY(Uall.alloc(sizeof(float) * (size_t)uofs[(size_t)nb], s));
    if (nlane == 1) {
        for (const auto &b : batches)
            HGM_TRY(run_batch(models, b.first, b.second, scene, params, offsets, n_lo, n_hi, Ed, Ad, zb.as<int64_t>(),
                              Mmax, s, 0, Uall.as<float>() + uofs[(size_t)(&b - batches.data())]));
    } else {
        cudaEvent_t fork = nullptr, join[MAX_LANES] = {};
        HGM_CUDA(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
        HGM_CUDA(cudaEventRecord(fork, s));
        hgm_status st = HGM_OK;
        for (int l = 0; l < nlane; ++l) HGM_CUDA(cudaStreamWaitEvent(aux_stream(scene->device, 1 + l), fork, 0));
        // lane l enqueues batches l, l + nlane, ... on its stream, each lane from its own host
        // thread (LanePool); a failing lane stops, its status and message are handed back
        std::vector<hgm_status> lst((size_t)nlane, HGM_OK);
        std::vector<std::string> lmsg((size_t)nlane);
        const int dev = scene->device;
        lane_pool().run(nlane, [&](int l) {
            cudaSetDevice(dev);
            for (int bi = l; bi < nb; bi += nlane) {
                const hgm_status bs = run_batch(models, batches[bi].first, batches[bi].second, scene, params, offsets,
                                                n_lo, n_hi, Ed, Ad, zb.as<int64_t>() + zlane * l, Mmax,
                                                aux_stream(dev, 1 + l), 1 + l, Uall.as<float>() + uofs[(size_t)bi]);
                if (bs != HGM_OK) {
                    lst[(size_t)l] = bs;
                    lmsg[(size_t)l] = g_err;
                    break;
                }
            }
        });
        for (int l = 0; l < nlane && st == HGM_OK; ++l)
            if (lst[(size_t)l] != HGM_OK) st = fail(lst[(size_t)l], lmsg[(size_t)l]);
        for (int l = 0; l < nlane; ++l) {  // join (also after a failure: nothing may outlive the call's buffers)
            cudaEventCreateWithFlags(&join[l], cudaEventDisableTiming);
            cudaEventRecord(join[l], aux_stream(scene->device, 1 + l));
            cudaStreamWaitEvent(s, join[l], 0);
            cudaEventDestroy(join[l]);
        }
        cudaEventDestroy(fork);
        HGM_TRY(st);
    }
    scene->uses.record(s);
    for (int m = 0; m < n_models; ++m) models[m]->uses.record(s);
    return HGM_OK;
}

static hgm_status check_dictionary(const hgm_model *const *models, int32_t n_models, const hgm_scene *scene,
                                   const hgm_params *params, const hgm_offsets *offsets, int32_t score_mode) {
    if (!models || n_models <= 0) return fail(HGM_ERR_EMPTY_POINT_SET, "empty model dictionary");
    if (!scene) return fail(HGM_ERR_INVALID_ARGUMENT, "NULL scene");
    HGM_TRY(check_params(params, scene));
    HGM_TRY(check_offsets(offsets));
    if (score_mode != 0 && score_mode != 1) return fail(HGM_ERR_INVALID_ARGUMENT, "score_mode must be 0 or 1");
    for (int m = 0; m < n_models; ++m) {
        if (!models[m]) return fail(HGM_ERR_INVALID_ARGUMENT, "NULL model handle");
        if (models[m]->F != scene->F) return fail(HGM_ERR_DIMENSION_MISMATCH, "model and scene descriptor lengths differ");
    }
    return HGM_OK;
}

// per-offset argmin of S [n_models][count] into host-or-device outputs; S_all copied
// out when the caller's pointer is a host one (a device S_all is already S).
static hgm_status finish_detect(const float *S, int n_models, int count, float threshold, int32_t *winner,
                                float *score, float *S_all, bool dSall, cudaStream_t s) {
    DevBuf wdev, sdev;
    const bool hw = winner && !is_device_ptr(winner), hs = score && !is_device_ptr(score);
    if (hw) HGM_TRY(wdev.alloc(sizeof(int32_t) * count, s));
    if (hs) HGM_TRY(sdev.alloc(sizeof(float) * count, s));
    HGM_TRY(offset_argmin(S, n_models, count, threshold, hw ? wdev.as<int32_t>() : winner,
                          hs ? sdev.as<float>() : score, s));
    if (hw) HGM_CUDA(cudaMemcpyAsync(winner, wdev.p, sizeof(int32_t) * count, cudaMemcpyDeviceToHost, s));
    if (hs) HGM_CUDA(cudaMemcpyAsync(score, sdev.p, sizeof(float) * count, cudaMemcpyDeviceToHost, s));
    if (S_all && !dSall)
        HGM_CUDA(cudaMemcpyAsync(S_all, S, sizeof(float) * (size_t)n_models * count, cudaMemcpyDeviceToHost, s));
    if (hw || hs || (S_all && !dSall)) HGM_CUDA(cudaStreamSynchronize(s));
    HGM_CUDA(cudaGetLastError());
    return HGM_OK;
}

hgm_status hgm_detect_actions(const hgm_model *const *models, int32_t n_models, const hgm_scene *scene,
                              const hgm_params *params, const hgm_offsets *offsets, int32_t score_mode,
                              float threshold, int32_t *winner, float *score, float *E_all, void *stream) {
    NvtxRange nvtx_("hgm_detect_actions");
    HGM_TRY(check_dictionary(models, n_models, scene, params, offsets, score_mode));
    const int count = offsets->count;
    if (count == 0) return HGM_OK;
    cudaStream_t s = (cudaStream_t)stream;
    HGM_CUDA(cudaSetDevice(scene->device));
    DevBuf Eb, Ab;
    const bool dEall = E_all && is_device_ptr(E_all);
    HGM_TRY(Ab.alloc(sizeof(float) * (size_t)n_models * count, s));
    if (!dEall) HGM_TRY(Eb.alloc(sizeof(float) * (size_t)n_models * count, s));
    float *Ed = dEall ? E_all : Eb.as<float>();
    HGM_TRY(detect_scores(models, n_models, scene, params, offsets, Ed, Ab.as<float>(), s));
    if (score_mode == 0) return finish_detect(Ed, n_models, count, threshold, winner, score, E_all, dEall, s);
    HGM_TRY(finish_detect(Ab.as<float>(), n_models, count, threshold, winner, score, nullptr, false, s));
    if (E_all && !dEall) {  // E_all always holds E*
        HGM_CUDA(cudaMemcpyAsync(E_all, Ed, sizeof(float) * (size_t)n_models * count, cudaMemcpyDeviceToHost, s));
        HGM_CUDA(cudaStreamSynchronize(s));
    }
    return HGM_OK;
}

hgm_status hgm_detect_chains(const hgm_model *const *chains, int32_t n_chains, const int32_t *chain_model,
                             int32_t n_models, const hgm_scene *scene, const hgm_params *params,
                             const hgm_offsets *offsets, int32_t score_mode, float threshold, int32_t *winner,
                             float *score, float *S_all, void *stream) {
    NvtxRange nvtx_("hgm_detect_chains");
    HGM_TRY(check_dictionary(chains, n_chains, scene, params, offsets, score_mode));
    if (!chain_model) return fail(HGM_ERR_INVALID_ARGUMENT, "chain_model == NULL");
    if (n_models < 1) return fail(HGM_ERR_EMPTY_POINT_SET, "no models");
    std::vector<int32_t> first((size_t)n_models + 1, 0);
    for (int c = 0; c < n_chains; ++c) {
        if (chain_model[c] < 0 || chain_model[c] >= n_models) return fail(HGM_ERR_INVALID_ARGUMENT, "chain_model out of range");
        if (c > 0 && chain_model[c] < chain_model[c - 1])
            return fail(HGM_ERR_INVALID_ARGUMENT, "chains must be grouped by model (chain_model non-decreasing)");
        ++first[(size_t)chain_model[c] + 1];
    }
    for (int m = 0; m < n_models; ++m) {
        if (first[(size_t)m + 1] == 0) return fail(HGM_ERR_EMPTY_POINT_SET, "a model has no chain");
        first[(size_t)m + 1] += first[(size_t)m];
    }
    const int count = offsets->count;
    if (count == 0) return HGM_OK;
    cudaStream_t s = (cudaStream_t)stream;
    HGM_CUDA(cudaSetDevice(scene->device));
    DevBuf Eb, Ab, Sb, fb;
    HGM_TRY(Eb.alloc(sizeof(float) * (size_t)n_chains * count, s));
    HGM_TRY(Ab.alloc(sizeof(float) * (size_t)n_chains * count, s));
    HGM_TRY(detect_scores(chains, n_chains, scene, params, offsets, Eb.as<float>(), Ab.as<float>(), s));
    const bool dSall = S_all && is_device_ptr(S_all);
    if (!dSall) HGM_TRY(Sb.alloc(sizeof(float) * (size_t)n_models * count, s));
    float *Sd = dSall ? S_all : Sb.as<float>();
    HGM_TRY(fb.alloc(sizeof(int32_t) * first.size(), s));
    HGM_CUDA(cudaMemcpyAsync(fb.p, first.data(), sizeof(int32_t) * first.size(), cudaMemcpyHostToDevice, s));
    HGM_TRY(chain_mean(score_mode == 0 ? Eb.as<float>() : Ab.as<float>(), fb.as<int32_t>(), n_models, count, Sd, s));
    HGM_TRY(finish_detect(Sd, n_models, count, threshold, winner, score, S_all, dSall, s));
    HGM_CUDA(cudaStreamSynchronize(s));  // `first` (host) must outlive its upload
    return HGM_OK;
}

hgm_status hgm_classify_blocks(const hgm_model *const *prototypes, int32_t n_prototypes, const int32_t *label,
                               int32_t n_labels, const hgm_scene *scene, const hgm_params *params,
                               const hgm_offsets *blocks, float threshold, int32_t *block_label, float *block_score,
                               int32_t *clip_label, void *stream) {
    NvtxRange nvtx_("hgm_classify_blocks");
    if (!prototypes || !scene || !params || !blocks) return fail(HGM_ERR_INVALID_ARGUMENT, "NULL argument");
    if (n_prototypes < 1) return fail(HGM_ERR_EMPTY_POINT_SET, "empty prototype dictionary");
    if (!label) return fail(HGM_ERR_INVALID_ARGUMENT, "label == NULL");
    if (n_labels < 1 || n_labels > 4096) return fail(HGM_ERR_INVALID_ARGUMENT, "n_labels must be 1..4096");
    for (int m = 0; m < n_prototypes; ++m)
        if (label[m] < 0 || label[m] >= n_labels) return fail(HGM_ERR_INVALID_ARGUMENT, "label out of range");
    HGM_TRY(check_offsets(blocks));
    const int count = blocks->count;
    cudaStream_t s = (cudaStream_t)stream;
    HGM_CUDA(cudaSetDevice(scene->device));
    DevBuf win, sco, lab, bl, cl;
    HGM_TRY(win.alloc(sizeof(int32_t) * std::max(count, 1), s));
    const bool hs = block_score && !is_device_ptr(block_score);
    if (hs || !block_score) HGM_TRY(sco.alloc(sizeof(float) * std::max(count, 1), s));
    float *sd = (hs || !block_score) ? sco.as<float>() : block_score;
    HGM_TRY(hgm_detect_actions(prototypes, n_prototypes, scene, params, blocks, /*score_mode=*/1, threshold,
                               win.as<int32_t>(), sd, nullptr, stream));
    HGM_TRY(lab.alloc(sizeof(int32_t) * n_prototypes, s));
    HGM_CUDA(cudaMemcpyAsync(lab.p, label, sizeof(int32_t) * n_prototypes, cudaMemcpyHostToDevice, s));
    const bool hb = block_label && !is_device_ptr(block_label), hc = clip_label && !is_device_ptr(clip_label);
    if (hb) HGM_TRY(bl.alloc(sizeof(int32_t) * std::max(count, 1), s));
    if (hc) HGM_TRY(cl.alloc(sizeof(int32_t), s));
    HGM_TRY(block_vote(win.as<int32_t>(), count, lab.as<int32_t>(), n_labels, hb ? bl.as<int32_t>() : block_label,
                       hc ? cl.as<int32_t>() : clip_label, s));
    HGM_CUDA(cudaGetLastError());
    if (hb) HGM_CUDA(cudaMemcpyAsync(block_label, bl.p, sizeof(int32_t) * count, cudaMemcpyDeviceToHost, s));
    if (hc) HGM_CUDA(cudaMemcpyAsync(clip_label, cl.p, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    if (hs) HGM_CUDA(cudaMemcpyAsync(block_score, sco.p, sizeof(float) * count, cudaMemcpyDeviceToHost, s));
    HGM_CUDA(cudaStreamSynchronize(s));  // the label array (host) and the scratch are released here
    return HGM_OK;
}

hgm_status hgm_set_profiling(int enable) {
    std::lock_guard<std::mutex> lk(g_mu);
    g_prof = enable != 0;
    while (g_prof && g_event_pool.size() < 1024) {  // pre-create: no event creation inside timed regions
        cudaEvent_t e = nullptr;
        if (cudaEventCreate(&e) != cudaSuccess) break;
        g_event_pool.push_back(e);
    }
    cudaGetLastError();
    return HGM_OK;
}

hgm_status hgm_get_stats(hgm_stats *out, int reset) {
    if (!out) return fail(HGM_ERR_INVALID_ARGUMENT, "out == NULL");
    std::lock_guard<std::mutex> lk(g_mu);
    for (auto &pe : g_pending) {
        float ms = 0.f;
        cudaEventSynchronize(pe.b);
        cudaEventElapsedTime(&ms, pe.a, pe.b);
        g_stats.ms[pe.cls] += ms;
        g_event_pool.push_back(pe.a);
        g_event_pool.push_back(pe.b);
    }
    g_pending.clear();
    *out = g_stats;
    if (reset) {
        g_stats = hgm_stats{};
        for (int k = 0; k < HP_NSLOT; ++k) g_hp_us[k] = 0.0, g_hp_n[k] = 0;  // (the host profile restarts too)
    }
    return HGM_OK;
}

}  // extern "C"
