// driver.cu -- host orchestration of one model batch at every offset:
// window descriptors, the frame tiling of K-DP's work items, chunking of the
// alpha history, one K-DP launch per recursion step i = M..3 (Eq. 10, the
// paper's host loop of Alg. 2 with the whole batch of windows per launch), then K-BT.
#include <algorithm>
#include <cstdio>
#include <memory>
#include <cstdlib>
#include <cstring>

#include "dp_common.cuh"

namespace hgm {

hgm_status launch_item_prep(const SceneView &v, const WorkItem *items, int nitems, const TileCaps &caps, int T,
                            unsigned char *book, cudaStream_t s);
size_t item_book_bytes(const TileCaps &caps, int T);
size_t item_stage_bytes(int NE, int NTH, int NC, int NA, int NB, int FT, int T, int NM, int book);
hgm_status launch_dp_batch(int NM, const SceneView &v, const WorkItem *items, int nitems, const unsigned char *book,
                           int *counter, float *hist, int64_t L, int layer, bool has_next, bool has_prev,
                           const StepConstB &kc, const float *U, int64_t ui_off, const DPParams &p,
                           const TileCaps &caps, cudaStream_t s, bool pdl_ok);
hgm_status launch_items(const SceneView &v, const InstDesc *dinst, int ninst, int W, int T, const int32_t *gstart,
                        const int32_t *tile_of, int tf_lo, const int32_t *sub_begin, const int32_t *sub_g,
                        const int32_t *item_base, int base0, WorkItem *items, cudaStream_t s);
hgm_status launch_init_ee(const InstDesc *dinst, int ninst, float *hist, int64_t L, int layer, int NM,
                          cudaStream_t s);
size_t dp_batch_smem(const TileCaps &c, int T, int NM);
hgm_status launch_backtrack_warp(const SceneView &v, const InstDesc *dinst, int ninst, const float *hist, int64_t L,
                                 const BTArgs &bt, const DPParams &p, cudaStream_t s);
hgm_status launch_dp_v0(const SceneView &v, const InstDesc *dinst, int ninst, int64_t maxNs, float *hist, int64_t L,
                        int layer, bool has_next, const StepConst &kc, const float *U, int64_t n_lo, const DPParams &p,
                        cudaStream_t s);
hgm_status launch_backtrack_v0(const SceneView &v, const InstDesc *dinst, int ninst, const float *hist, int64_t L,
                               const BTArgs &bt, const DPParams &p, cudaStream_t s);
hgm_status launch_dp_window(int NM, const SceneView &v, const InstDesc *dinst, int ninst, float *hist, int64_t L,
                            int M, const WinStepPtrs &sp, const float *U, int64_t nn, int64_t n_lo,
                            const DPParams &p, const WinCaps &caps, cudaStream_t s);
size_t dp_window_smem(const WinCaps &c, int NM);

static inline int host_first(const hgm_scene *sc, int64_t f) {
    if (f <= 0) return 0;
    if (f > sc->fmax) return (int)sc->S;
    return sc->first_h[f];
}

// extra streams per device: index 0 = the second lane of the chunk pipeline, 1.. = the
// lanes of concurrent model batches (detect_scores)
constexpr int N_AUX = 1 + MAX_LANES;
cudaStream_t aux_stream(int device, int idx) {
    static std::mutex mu;
    static cudaStream_t as[64][N_AUX] = {};
    std::lock_guard<std::mutex> lk(mu);
    if (device < 0 || device >= 64 || idx < 0 || idx >= N_AUX) return nullptr;
    if (!as[device][idx]) cudaStreamCreateWithFlags(&as[device][idx], cudaStreamNonBlocking);
    return as[device][idx];
}

// Per-device cache of K-DP's large scratch buffers (alpha history, work items, item
// bookkeeping, counters).  Allocating gigabytes per call from the stream-ordered pool maps
// fresh pages whenever the previous call's free is not yet known complete on the new
// call's stream (host-API calls use a fresh stream each), which made calls erratic.  A
// call waits for the previous user's work (event) before touching the buffers and
// records its own completion; buffers only grow.
struct Scratch {
    void *p = nullptr;
    size_t cap = 0;
    hgm_status ensure(size_t bytes) {
        if (bytes <= cap) return HGM_OK;
        if (p) cudaFree(p);  // synchronous, but rare (growth only)
        p = nullptr;
        cap = 0;
        const size_t want = bytes + bytes / 4;
        if (cudaMalloc(&p, want) != cudaSuccess) {
            cudaGetLastError();
            if (cudaMalloc(&p, bytes) != cudaSuccess) {
                p = nullptr;
                return cuda_fail(cudaGetLastError(), "cudaMalloc(K-DP scratch)");
            }
            cap = bytes;
            return HGM_OK;
        }
        cap = want;
        return HGM_OK;
    }
};
// Pinned host staging for a call's small uploads (window descriptors, item prefixes, frame
// tiling): a copy from pageable memory is staged by the driver and can block the host for
// tens of microseconds, which dominated the enqueue of few-window calls (50-model context
// rows: 0.41 of 0.69 ms was host enqueue, tools/ctx_probe.py).  The buffer is reused once the
// previous call's copies have read it (event).
struct PinnedStage {
    char *p = nullptr;
    size_t cap = 0, used = 0;
    cudaEvent_t read = nullptr;  // the last call's copies out of the buffer completed
    hgm_status begin(size_t bytes) {
        if (read) HGM_CUDA(cudaEventSynchronize(read));
        else HGM_CUDA(cudaEventCreateWithFlags(&read, cudaEventDisableTiming));
        if (bytes > cap) {
            if (p) cudaFreeHost(p);
            p = nullptr;
            cap = 0;
            const size_t want = std::max<size_t>(bytes, (size_t)1 << 16);
            HGM_CUDA(cudaMallocHost(&p, want));
            cap = want;
        }
        used = 0;
        return HGM_OK;
    }
    // copy host bytes into the buffer and enqueue their transfer to dst on s
    hgm_status put(void *dst, const void *src, size_t bytes, cudaStream_t s) {
        if (!bytes) return HGM_OK;
        memcpy(p + used, src, bytes);
        HGM_CUDA(cudaMemcpyAsync(dst, p + used, bytes, cudaMemcpyHostToDevice, s));
        used += (bytes + 15) & ~(size_t)15;
        return HGM_OK;
    }
    hgm_status end(cudaStream_t s) {
        HGM_CUDA(cudaEventRecord(read, s));
        return HGM_OK;
    }
};

struct ScratchSet {
    std::mutex mu;
    Scratch hist, items, book, counters, desc;
    cudaEvent_t done = nullptr;
    PinnedStage up;
};
// one set per (device, lane): lane 0 serves single-batch calls, lanes 1.. the concurrent
// model batches of a detect call (each lane is one stream, so its set is never shared)
static ScratchSet &scratch_set(int device, int lane) {
    static std::mutex mu;
    static ScratchSet *sets[64][MAX_LANES + 1] = {};
    std::lock_guard<std::mutex> lk(mu);
    const int d = device < 0 || device >= 64 ? 0 : device;
    const int l = lane < 0 || lane > MAX_LANES ? 0 : lane;
    if (!sets[d][l]) sets[d][l] = new ScratchSet();
    return *sets[d][l];
}

// device memory size, read once per device (cudaMemGetInfo per call cost ~0.25 ms of host
// time on small calls: the single 754-node instance went 0.35 -> 0.60 ms)
static size_t device_total_mem(int device) {
    static std::mutex mu;
    static size_t total[64] = {};
    const int d = device < 0 || device >= 64 ? 0 : device;
    std::lock_guard<std::mutex> lk(mu);
    if (!total[d]) {
        size_t fr = 0, tot = 0;
        total[d] = cudaMemGetInfo(&fr, &tot) == cudaSuccess && tot > 0 ? tot : ((size_t)96 << 30);
        cudaGetLastError();
    }
    return total[d];
}

thread_local bool g_tiling_failed = false;

bool use_v0_kernels() {
    const char *e = getenv("HGM_KERNEL");
    return e && strcmp(e, "v0") == 0;
}

// K-DP tiling: the frames [f_lo, f_hi) the call's windows cover are cut into tiles
// of consecutive b-frames, greedily: a tile grows while the shared-memory footprint
// of its two big buffers (candidate entries + raw alpha rows, 2 stages of direction
// rows) stays under a cap; a single frame is always a tile.  A window's work items
// are the tiles meeting its frames, clipped to them.  The kernel's shared-memory
// plan is sized to the maxima over the tiles produced; the cap shrinks until the
// plan fits the budget (2 CTAs per SM), else a 1-CTA-per-SM budget is tried.
struct Tiling {
    TileCaps caps{};
    std::vector<int32_t> gstart;     // b-tile start frames, then f_hi, then sentinels
    std::vector<int32_t> tile_of;    // b-tile index of frame f_lo + q
    std::vector<int32_t> sub_begin;  // a-frame chunks of b-tile q: [sub_begin[q], sub_begin[q+1])
    std::vector<int32_t> sub_g;      // chunk j covers a-frames [sub_g[2j], sub_g[2j+1])
    int f_lo = 0;
    // work items of the window starting at frame `of` (the same rule as k_items)
    int items_of(int64_t of, int W) const {
        int n = 0;
        for (int gt = tile_of[of - f_lo]; gt <= tile_of[of + W - 1 - f_lo]; ++gt) {
            const int64_t F1 = std::min<int64_t>(gstart[gt + 1], of + W);
            bool first = true;
            for (int sb = sub_begin[gt]; sb < sub_begin[gt + 1]; ++sb) {
                const int64_t G0 = std::max<int64_t>(sub_g[2 * sb], of), G1 = std::min<int64_t>(sub_g[2 * sb + 1], F1);
                if (G0 >= G1 && !first) continue;
                first = false;
                ++n;
            }
        }
        return n;
    }
};

static bool make_tiling(const hgm_scene *sc, const hgm_offsets &o, int T, int NM, Tiling *tl) {
    const int64_t f_lo = o.first_frame;
    const int64_t f_hi = (int64_t)o.first_frame + (int64_t)(o.count - 1) * o.stride + o.window;
    auto QP = [&](int64_t f) { return (int64_t)sc->qpad_h[host_first(sc, f)]; };
    auto NF = [&](int64_t f) { return (int64_t)host_first(sc, f); };
    const int FT_max = std::max(1, std::min(8, 255 / std::max(1, T - 1)));
    const char *benv = getenv("HGM_SMEM_KB");  // tuning knob: shared memory per CTA (2 CTAs per SM by default)
    // (shared-memory budget, stages): 2 CTAs/SM double-buffered; 1 CTA/SM double-buffered;
    // 1 CTA/SM single stage (items too large for two, i.e. large T)
    const char *nenv = getenv("HGM_STAGES");  // tuning knob: stages of the first budget (2 or 3)
    size_t budgets[3] = {(size_t)(benv ? atoi(benv) : 110) * 1024, 220 * 1024, 220 * 1024};
    if (const char *menv = getenv("HGM_SMEM_MAX_KB"))  // testing: cap every budget (forces the fallbacks)
        for (size_t &b : budgets) b = std::min(b, (size_t)atoi(menv) * 1024);
    int stages[3] = {nenv ? std::max(1, std::min(3, atoi(nenv))) : 2, 2, 1};
    if (getenv("HGM_SINGLE_STAGE"))  // testing: every budget single-staged (the large-T fallback path)
        stages[0] = stages[1] = 1;
    if (T > 128 && !benv && !nenv) {
        // b-tiles are single frames here (FT_max = 1) and items are a-frame chunks whose
        // fixed part (b-row entries, row tables) is amortised over the chunk: one single
        // stage per CTA.  One 220 KB stage per SM measured faster than two 110 KB stages or
        // two 220 KB ones before task splitting and programmatic dependent launch (single
        // instance, T = 320: 7.3 -> 4.7 ms); with them, two CTAs per SM with one 110 KB
        // stage each are faster again (T = +inf: 8.17 -> 7.47 ms, profiles/r02b/r02al_*)
        budgets[0] = std::min(budgets[2], (size_t)110 * 1024);
        stages[0] = 1;
    }
    // stage bytes of the unclipped item: b-frames [a, b), a-frames [g0, g1)
    auto foot = [&](int64_t a, int64_t b, int64_t g0, int64_t g1, int64_t book) {
        const int64_t nrows = std::min(NF(g1), NF(a)) - NF(g0) + (NF(b) - NF(a));  // a rows before the b rows + b rows
        return (int64_t)item_stage_bytes((int)(QP(b) - QP(a)), (int)(QP(g1) - QP(g0)), (int)(NF(b + T - 1) - NF(a)),
                                         (int)nrows, (int)(NF(b) - NF(a)), (int)(b - a), T, NM, (int)book);
    };
    for (int bi = 0; bi < 3; ++bi) {
        TileCaps c0{1, 1, 1, 1, 1, 1, FT_max, o.window, 0, stages[bi]};
        const int64_t fixed = (int64_t)dp_batch_smem(c0, T, NM);  // stage-independent part (upper bound)
        const int64_t cap = ((int64_t)budgets[bi] - fixed) / stages[bi] / 16 * 16;
        TileCaps cb{1, 1, 1, 1, 1, 1, 1, o.window, 0, stages[bi]};
        int64_t book = (int64_t)item_book_bytes(cb, T);  // grows below until it covers the tiles made with it
        for (int iter = 0; iter < 6; ++iter) {
            Tiling t;
            t.f_lo = (int)f_lo;
            TileCaps c{1, 1, 1, 1, 1, 1, 1, o.window, 0, stages[bi]};
            bool fits = true;
            auto account = [&](int64_t F0, int64_t F1, int64_t G0, int64_t G1) {
                c.STAGE = (int)std::max<int64_t>(c.STAGE, foot(F0, F1, G0, G1, book));
                c.NE = (int)std::max<int64_t>(c.NE, QP(F1) - QP(F0));
                c.TH = (int)std::max<int64_t>(c.TH, QP(G1) - QP(G0) + 8);
                c.NA = (int)std::max<int64_t>(c.NA, std::min(NF(G1), NF(F0)) - NF(G0) + NF(F1) - NF(F0));
                c.NB = (int)std::max<int64_t>(c.NB, NF(F1) - NF(F0));
                c.NC = (int)std::max<int64_t>(c.NC, NF(F1 + T - 1) - NF(F0));
                int64_t nst = 0;
                for (int64_t f = F0; f < F1; ++f)
                    nst += (NF(f + 1) - NF(f)) * (NF(std::min(f, G1)) - NF(std::max(f - T + 1, G0)));
                c.NST = (int)std::max<int64_t>(c.NST, nst);
                c.FT = (int)std::max<int64_t>(c.FT, F1 - F0);
                t.sub_g.push_back((int32_t)G0);
                t.sub_g.push_back((int32_t)G1);
            };
            for (int64_t F0 = f_lo; F0 < f_hi && fits;) {
                int64_t F1 = F0 + 1;  // a single frame is always a b-tile
                while (F1 < f_hi && F1 - F0 < FT_max && foot(F0, F1 + 1, F0 - T + 1, F1 + 1, book) <= cap) ++F1;
                t.gstart.push_back((int32_t)F0);
                t.sub_begin.push_back((int32_t)(t.sub_g.size() / 2));
                if ((F1 - F0) * (T - 1) <= 255 && foot(F0, F1, F0 - T + 1, F1, book) <= cap) {
                    account(F0, F1, F0 - T + 1, F1);  // one item covers every a-frame
                } else {  // large T (only a single b-frame gets here): its a-frames [F0 - T + 1, F1) in chunks
                    for (int64_t G0 = F0 - T + 1; G0 < F1 && fits;) {
                        int64_t G1 = G0 + 1;
                        if (foot(F0, F1, G0, G1, book) > cap) fits = false;
                        // largest G1 <= F1 whose item fits: <= 255 segments (k_item_prep's uint8
                        // state -> segment map) and the stage cap; both monotone in G1, so a
                        // binary search finds what growing G1 one frame at a time would
                        if (fits) {
                            int64_t lo = G1, hi = F1;
                            while (lo < hi) {
                                const int64_t mid = (lo + hi + 1) / 2;
                                if ((mid - G0) * (F1 - F0) <= 255 && foot(F0, F1, G0, mid, book) <= cap)
                                    lo = mid;
                                else
                                    hi = mid - 1;
                            }
                            G1 = lo;
                        }
                        account(F0, F1, G0, G1);
                        G0 = G1;
                    }
                }
                F0 = F1;
            }
            if (!fits) break;  // a single (b-frame, a-frame) item exceeds this budget
            const int64_t need_book = (int64_t)item_book_bytes(c, T);
            if (need_book > book) {  // the bookkeeping record grew: retile with it
                book = need_book;
                continue;
            }
            if (c.STAGE > cap || dp_batch_smem(c, T, NM) > budgets[bi]) break;
            const int ntiles = (int)t.gstart.size();
            t.gstart.push_back((int32_t)f_hi);
            t.sub_begin.push_back((int32_t)(t.sub_g.size() / 2));
            t.tile_of.resize((size_t)(f_hi - f_lo));
            for (int q = 0; q < ntiles; ++q)
                for (int64_t f = t.gstart[q]; f < t.gstart[q + 1]; ++f) t.tile_of[f - f_lo] = q;
            t.gstart.push_back(INT32_MAX / 2);
            t.sub_begin.push_back(t.sub_begin.back());
            c.STAGE = (int)std::max<int64_t>(c.STAGE, 16);
            if (getenv("HGM_DEBUG_TILING"))  // diagnosis
                fprintf(stderr, "tiling: NM %d budget %zu stages %d cap %lld tiles %d subs %zu STAGE %d NE %d TH %d NA %d NB %d NC %d NST %d smem %zu\n",
                        NM, budgets[bi], stages[bi], (long long)cap, ntiles, t.sub_g.size() / 2, c.STAGE, c.NE, c.TH,
                        c.NA, c.NB, c.NC, c.NST, dp_batch_smem(c, T, NM));
            t.caps = c;
            *tl = std::move(t);
            return true;
        }
    }
    return false;
}

// K-DPW eligibility: the largest window of the call (its padded band, nodes, task list)
// must fit one CTA's shared memory.  Tasks per window are counted exactly from the frame
// histogram (one task = a b with a pair of a's of one frame).  HGM_DP=fused / window
// forces a path (the window path still needs to fit).
static bool window_path(const hgm_scene *sc, const std::vector<InstDesc> &all, int NM, const hgm_offsets &o, int T,
                        int M, WinCaps *caps) {
    const char *e = getenv("HGM_DP");
    if (e && strcmp(e, "fused") == 0) return false;
    WinCaps c{0, 0, o.window, 0, T, M};
    for (const InstDesc &d : all) {
        c.NPP = std::max(c.NPP, d.npp);
        c.SW = std::max(c.SW, d.we - d.wb);
    }
    if (c.SW >= 32768) return false;  // tasks pack node indices in 15 / 16 bits
    // a handful of LARGE windows: one CTA per window would leave the GPU idle where the
    // per-step kernel spreads each step over every SM (one 754-node window, T = 10:
    // 0.45 ms on K-DPW vs 0.26 ms fused)
    if (!(e && strcmp(e, "window") == 0) && all.size() < 4 && c.NPP > 2048) return false;
    const size_t limit = 227 * 1024;
    if (dp_window_smem(c, NM) > limit) return false;  // even without a task list
    // tasks of the busiest window, bounded from the frame histogram: per b-frame fb,
    // n(fb) * sum_g ceil(n(fb - g) / 2) (every gap, ignoring the clip at the window start),
    // summed over the window's frames by a prefix sum -- O(frames x T + windows)
    const int64_t f_lo = all.front().o, f_hi = (int64_t)all.back().o + o.window;
    std::vector<int64_t> pre((size_t)(f_hi - f_lo) + 1, 0);
    auto nfr = [&](int64_t f) { return (int64_t)host_first(sc, f + 1) - host_first(sc, f); };
    for (int64_t fb = f_lo; fb < f_hi; ++fb) {
        const int64_t nb = nfr(fb);
        int64_t t = 0;
        if (nb)
            for (int g = 1; g < T; ++g) t += (nfr(fb - g) + 1) / 2;
        pre[(size_t)(fb - f_lo) + 1] = pre[(size_t)(fb - f_lo)] + nb * t;
    }
    int64_t ntask_max = 0;
    for (const InstDesc &d : all)
        ntask_max = std::max(ntask_max, pre[(size_t)(d.o + o.window - f_lo)] - pre[(size_t)(d.o - f_lo)]);
    c.NTASK = (int)std::max<int64_t>(1, ntask_max);
    if (dp_window_smem(c, NM) > limit) return false;
    *caps = c;
    return true;
}

// Match NM models of equal chain length M at every offset.
// U: batched unary table U[((i * nn) + (n - n_lo)) * NM + k].
hgm_status match_batch(const hgm_model *const *models, int NM, const hgm_scene *sc, const hgm_params &pp,
                       const hgm_offsets &o, const float *U, const float *Us, int64_t n_lo, int64_t nn,
                       const MatchOut *outs, cudaStream_t s, int lane) {
    std::unique_ptr<HostPhase> hp(new HostPhase(HP_PLAN));
    const int count = o.count, M = models[0]->M;
    if (count <= 0) return HGM_OK;
    if (NM < 1 || NM > MAX_BATCH) return fail(HGM_ERR_INVALID_ARGUMENT, "model batch size must be 1..8");
    bool v0 = use_v0_kernels();
    if (v0 && NM != 1) return fail(HGM_ERR_INVALID_ARGUMENT, "v0 kernels take one model at a time");
    const int nsteps = M >= 3 ? M - 2 : 0;
    std::vector<InstDesc> all(count);
    for (int k = 0; k < count; ++k) {
        const int64_t of = (int64_t)o.first_frame + (int64_t)k * o.stride;
        InstDesc d{};
        d.wb = host_first(sc, of);
        d.we = host_first(sc, of + o.window);
        d.pbase = sc->qstart_h[d.wb];
        d.np = sc->qstart_h[d.we] - sc->qstart_h[d.wb];
        d.ppad = sc->qpad_h[d.wb];
        d.npp = sc->qpad_h[d.we] - sc->qpad_h[d.wb];
        d.ntail = d.npp;
        d.out = k;
        d.o = (int32_t)of;
        all[k] = d;
    }
    WinCaps wcaps{};
    const bool win = !v0 && nsteps > 0 && window_path(sc, all, NM, o, pp.T, M, &wcaps);
    if (win && getenv("HGM_DEBUG_TILING"))
        fprintf(stderr, "window kernel: NM %d NPP %d SW %d NTASK %d smem %zu windows %d\n", NM, wcaps.NPP, wcaps.SW,
                wcaps.NTASK, dp_window_smem(wcaps, NM), count);
    Tiling tl;
    if (!v0 && !win && !make_tiling(sc, o, pp.T, NM, &tl)) {
        // a single (b-frame, a-frame) item of these frames exceeds shared memory (very
        // dense frames at large T): a batch is retried one model at a time by the caller,
        // and a single model falls back to the reference kernels (global-memory operands)
        if (getenv("HGM_DEBUG_TILING")) fprintf(stderr, "tiling: NM %d does not fit%s\n", NM, NM > 1 ? "" : ": v0 fallback");
        if (NM > 1) {
            g_tiling_failed = true;
            return fail(HGM_ERR_INVALID_ARGUMENT, "frames too dense for the shared-memory tile of a model batch");
        }
        v0 = true;
    }
    if (v0)
        for (InstDesc &d : all) d.ntail = d.np;  // v0 kernels: compact pair layout
    DPParams p;
    p.l1 = pp.lambda1;
    p.l2 = pp.lambda2;
    p.l23 = pp.lambda2 * pp.lambda3;  // one IEEE single multiply
    p.W = pp.w_dummy;
    p.l1W = pp.lambda1 * pp.w_dummy;
    p.T = pp.T;
    const SceneView v{sc->t,    sc->first_tab, sc->qstart,    sc->theta,    sc->coinc, sc->cpre,
                      sc->prow, sc->id,        sc->qpad,      sc->theta_pad, sc->prow_pad, sc->rfc,
                      sc->rlc,  sc->ninfo,     sc->fmax,      (int)sc->S};
    // Windows are processed in chunks: the alpha history of a chunk (every layer) must fit
    // the budget.  Larger chunks amortise each step launch's tail and each chunk's backtrack
    // over more windows (A/B on one B200, profiles/r02b/r02ag_hist_budget_ab.txt: C3 338.4 ->
    // 321.9 ms from 6 to 24 GiB, C2 -4.5 %, C4 T=20 -5 %; 48 GiB a further -0.7 %); a layer of
    // a C3 chunk is far larger than L2 either way.  Budget: min(24 GiB, 1/6 of the device's
    // memory); HGM_HIST_GB overrides (tuning).  Optionally chunks alternate between two streams.
    const char *genv = getenv("HGM_HIST_GB");
    // ... except for calls whose chunks hold few windows (the two-chunk-lane regime below,
    // judged at 6 GiB chunks): those keep >= 12 chunks (budget >= 6 GiB) so the two lanes
    // pipeline -- a handful of big chunks leaves the last one running alone (C4 T=20 rho=2:
    // 226 -> 281 ms with 24 GiB chunks; C2, one lane, 304 -> 290 ms)
    int64_t hist_total = 0;
    {
        const int SSb = v0 ? 1 : (win ? NM : entry_floats(NM));
        for (const InstDesc &d : all) {
            const int64_t ns = (int64_t)d.ntail + 2 * (int64_t)(d.we - d.wb) + 1;
            hist_total += (win ? (ns * SSb + 3) & ~(int64_t)3 : ns * SSb) * std::max(nsteps, 1);
        }
    }
    int64_t budget_floats = std::min<int64_t>((int64_t)24 << 28, (int64_t)(device_total_mem(sc->device) / 6 / sizeof(float)));
    {
        const int64_t n6 = (hist_total + ((int64_t)6 << 28) - 1) / ((int64_t)6 << 28);  // chunks at 6 GiB
        if (n6 >= 3 && (int64_t)count < 64 * n6)
            budget_floats = std::min(budget_floats, std::max<int64_t>((int64_t)6 << 28, hist_total / 12));
    }
    if (genv && atoi(genv) > 0) budget_floats = (int64_t)atoi(genv) << 28;
    BTArgs bt{};
    bt.U = U;
    bt.Us = Us;
    bt.nn = nn;
    bt.n_lo = n_lo;
    bt.NM = NM;
    bt.M = M;
    // floats per state in a layer: entry_floats(NM) for K-DP's 16-byte bulk copies, NM for
    // K-DPW (whole layers are 16-byte aligned instead), 1 for the v0 kernels
    const int SS = v0 ? 1 : (win ? NM : entry_floats(NM));
    bt.SS = SS;
    for (int k = 0; k < NM; ++k) {
        bt.step[k] = models[k]->step;
        bt.E[k] = outs[k].E;
        bt.A[k] = outs[k].A;
        bt.z[k] = outs[k].z;
    }
    const char *cenv = getenv("HGM_CHUNK");  // windows per chunk (tuning knob)
    const int chunk_max = std::min(65535, cenv && atoi(cenv) > 0 ? atoi(cenv) : 4096);
    // Chunks of windows (the alpha history of a chunk fits the budget), every window's
    // layer offset and work-item count, planned up front so that the window
    // descriptors and item prefixes reach the device in one copy each (no per-chunk
    // pageable copies between the chunks' kernels).
    struct Chunk {
        int k0, k1, nitems;
        int64_t L, maxNs;
    };
    std::vector<Chunk> chunks;
    std::vector<int32_t> ibase_all((size_t)count + 1, 0);
    int64_t max_hist = 4, max_items = 1;
    for (int k0 = 0; k0 < count;) {
        Chunk c{k0, k0, 0, 0, 1};
        while (c.k1 < count && c.k1 - k0 < chunk_max) {
            InstDesc &d = all[c.k1];
            const int64_t ns = (int64_t)d.ntail + 2 * (int64_t)(d.we - d.wb) + 1;
            const int64_t lw = win ? (ns * SS + 3) & ~(int64_t)3 : ns * SS;  // K-DPW: 16-byte aligned layers
            if (c.k1 > k0 && (c.L + lw) * std::max(nsteps, 1) > budget_floats) break;
            d.off = c.L;
            c.L += lw;
            c.maxNs = std::max(c.maxNs, ns);
            if (!v0 && !win) ibase_all[c.k1 + 1] = ibase_all[c.k1] + tl.items_of(d.o, o.window);
            ++c.k1;
        }
        c.nitems = ibase_all[c.k1] - ibase_all[k0];
        max_hist = std::max(max_hist, c.L * nsteps + 4);  // + 16 bytes: K-DP's bulk copies round to 16-byte units
        max_items = std::max<int64_t>(max_items, c.nitems);
        chunks.push_back(c);
        k0 = c.k1;
    }
    // Two lanes (chunks alternate over two streams, each with its own buffers) when the
    // chunks are few-window ones (long chains / wide windows: C4): a chunk's last DP
    // steps and its backtrack leave the GPU mostly idle, the other lane fills it
    // (C4, ~8 windows per chunk: 21-32 % less time per call).  Many-window chunks (C3,
    // ~3,200 per 24 GiB chunk) are faster on one lane, and a second lane doubles the history.
    const char *senv = getenv("HGM_STREAMS");  // 1 / 2: force
    const int nlanes = lane > 0 ? 1  // a concurrent model batch: its lane is the only one
                                : senv ? (atoi(senv) == 2 ? 2 : 1)
                                       : ((chunks.size() >= 3 && (int64_t)count < 64 * (int64_t)chunks.size()) ? 2 : 1);
    struct Lane {
        cudaStream_t s = nullptr;
        DevBuf hist, items, counters, book;
        int64_t hist_cap = 0, items_cap = 0, counters_cap = 0, book_cap = 0;
    } lanes[2];
    lanes[0].s = s;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    if (nlanes == 2) {
        lanes[1].s = aux_stream(sc->device, 0);
        HGM_CUDA(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
        HGM_CUDA(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
    }
    ScratchSet &scr = scratch_set(sc->device, lane);
    std::unique_lock<std::mutex> scr_lock(scr.mu);  // held while this call enqueues work on the buffers
    if (!scr.done) HGM_CUDA(cudaEventCreateWithFlags(&scr.done, cudaEventDisableTiming));
    HGM_CUDA(cudaStreamWaitEvent(s, scr.done, 0));  // the previous user's kernels are done with them
    hp.reset(new HostPhase(HP_UPLOAD));
    // the call's small device arrays (window descriptors, item prefixes, frame tiling) live in
    // the lane's cached descriptor scratch (no allocation per call) and are filled from its
    // pinned staging buffer
    InstDesc *d_all = nullptr;
    int32_t *d_ibase = nullptr, *d_subb = nullptr, *d_subg = nullptr, *d_gstart = nullptr, *d_tile_of = nullptr;
    {
        const bool tiled = !v0 && !win;
        auto rnd = [](size_t b) { return (b + 255) & ~(size_t)255; };
        const size_t b_all = rnd(sizeof(InstDesc) * count), b_ib = tiled ? rnd(4 * ((size_t)count + 1)) : 0,
                     b_sb = tiled ? rnd(4 * tl.sub_begin.size()) : 0,
                     b_sg = tiled ? rnd(4 * std::max<size_t>(2, tl.sub_g.size())) : 0,
                     b_gs = tiled ? rnd(4 * tl.gstart.size()) : 0,
                     b_to = tiled ? rnd(4 * std::max<size_t>(1, tl.tile_of.size())) : 0;
        HGM_TRY(scr.desc.ensure(b_all + b_ib + b_sb + b_sg + b_gs + b_to));
        char *q = static_cast<char *>(scr.desc.p);
        d_all = reinterpret_cast<InstDesc *>(q);
        q += b_all;
        if (tiled) {
            d_ibase = reinterpret_cast<int32_t *>(q);
            d_subb = reinterpret_cast<int32_t *>(q += b_ib);
            d_subg = reinterpret_cast<int32_t *>(q += b_sb);
            d_gstart = reinterpret_cast<int32_t *>(q += b_sg);
            d_tile_of = reinterpret_cast<int32_t *>(q += b_gs);
        }
        HGM_TRY(scr.up.begin(b_all + b_ib + b_sb + b_sg + b_gs + b_to + 96));
        HGM_TRY(scr.up.put(d_all, all.data(), sizeof(InstDesc) * count, s));
        if (tiled) {
            HGM_TRY(scr.up.put(d_ibase, ibase_all.data(), sizeof(int32_t) * (count + 1), s));
            HGM_TRY(scr.up.put(d_subb, tl.sub_begin.data(), sizeof(int32_t) * tl.sub_begin.size(), s));
            HGM_TRY(scr.up.put(d_subg, tl.sub_g.data(), sizeof(int32_t) * tl.sub_g.size(), s));
            HGM_TRY(scr.up.put(d_gstart, tl.gstart.data(), sizeof(int32_t) * tl.gstart.size(), s));
            HGM_TRY(scr.up.put(d_tile_of, tl.tile_of.data(), sizeof(int32_t) * tl.tile_of.size(), s));
        }
        HGM_TRY(scr.up.end(s));
    }
    if (nlanes == 2) {  // the second lane starts after the uploads
        HGM_CUDA(cudaEventRecord(ev_fork, s));
        HGM_CUDA(cudaStreamWaitEvent(lanes[1].s, ev_fork, 0));
    }
    hp.reset(new HostPhase(HP_DP));
    hgm_status st = HGM_OK;
    for (int chunk = 0; chunk < (int)chunks.size() && st == HGM_OK; ++chunk) {
        const Chunk &ch = chunks[chunk];
        Lane &ln = lanes[chunk % nlanes];
        const cudaStream_t ls = ln.s;
        const int k0 = ch.k0, ninst = ch.k1 - ch.k0;
        const int64_t L = ch.L, maxNs = ch.maxNs;
        cudaError_t e = cudaSuccess;
        float *hist = nullptr;
        if (chunk % nlanes == 0) {
            if ((st = scr.hist.ensure(sizeof(float) * max_hist)) != HGM_OK) break;
            hist = static_cast<float *>(scr.hist.p);
        } else {
            if (max_hist > ln.hist_cap) {
                if ((st = ln.hist.alloc(sizeof(float) * max_hist, ls)) != HGM_OK) break;
                ln.hist_cap = max_hist;
            }
            hist = ln.hist.as<float>();
        }
        const InstDesc *di = d_all + k0;
        const int nitems = ch.nitems;
        WorkItem *items_p = nullptr;
        int *counters_p = nullptr;
        unsigned char *book_p = nullptr;
        if (!v0 && !win && nsteps > 0) {
            const int64_t bbytes = (int64_t)item_book_bytes(tl.caps, p.T) * max_items + 16;
            if (chunk % nlanes == 0) {
                if ((st = scr.items.ensure(sizeof(WorkItem) * max_items)) != HGM_OK) break;
                if ((st = scr.counters.ensure(sizeof(int) * nsteps)) != HGM_OK) break;
                if ((st = scr.book.ensure(bbytes)) != HGM_OK) break;
                items_p = static_cast<WorkItem *>(scr.items.p);
                counters_p = static_cast<int *>(scr.counters.p);
                book_p = static_cast<unsigned char *>(scr.book.p);
            } else {
                if (max_items > ln.items_cap) {
                    if ((st = ln.items.alloc(sizeof(WorkItem) * max_items, ls)) != HGM_OK) break;
                    ln.items_cap = max_items;
                }
                if (nsteps > ln.counters_cap) {
                    if ((st = ln.counters.alloc(sizeof(int) * nsteps, ls)) != HGM_OK) break;
                    ln.counters_cap = nsteps;
                }
                if (bbytes > ln.book_cap) {
                    if ((st = ln.book.alloc(bbytes, ls)) != HGM_OK) break;
                    ln.book_cap = bbytes;
                }
                items_p = ln.items.as<WorkItem>();
                counters_p = ln.counters.as<int>();
                book_p = ln.book.as<unsigned char>();
            }
            HGM_CUDA(cudaMemsetAsync(counters_p, 0, sizeof(int) * nsteps, ls));
            launch_items(v, di, ninst, o.window, p.T, d_gstart, d_tile_of, tl.f_lo,
                         d_subb, d_subg, d_ibase + k0, ibase_all[k0], items_p,
                         ls);
            launch_item_prep(v, items_p, nitems, tl.caps, p.T, book_p, ls);
            launch_init_ee(di, ninst, hist, L, nsteps - 1, NM, ls);  // first layer's (eps, eps) slots
            count_launch(K_DP, 3);
        }
        // one timer around the chunk's consecutive K-DP launches (M-2 of them): nothing
        // else runs on the stream in between
        std::unique_ptr<Timer> dp_timer(nsteps > 0 ? new Timer(ls, K_DP) : nullptr);
        if (win && nsteps > 0) {  // K-DPW: every step of the chunk's windows in one launch
            WinStepPtrs sp{};
            for (int k = 0; k < NM; ++k) sp.step[k] = models[k]->step;
            st = launch_dp_window(NM, v, di, ninst, hist, L, M, sp, Us, nn, n_lo, p, wcaps, ls);
            count_launch(K_DP);
        }
        for (int i = M - 1; i >= 2 && st == HGM_OK && !win; --i) {
            const bool has_next = i + 1 <= M - 1;
            if (v0) {
                const float4 h = models[0]->step_h[i];
                const StepConst kc{h.x, h.y, h.z, h.w};
                st = launch_dp_v0(v, di, ninst, maxNs, hist, L, i - 2, has_next, kc, Us + (int64_t)i * nn, n_lo, p, ls);
                count_launch(K_DP);
                continue;
            }
            StepConstB kc{};
            for (int k = 0; k < NM; ++k) kc.c[k] = models[k]->step_h[i];
            for (int q = 0; q < (NM + 1) / 2; ++q) {
                const int k1 = std::min(2 * q + 1, NM - 1);
                kc.nA1[q] = make_float2(-kc.c[2 * q].z, -kc.c[k1].z);
                kc.nK2[q] = make_float2(-kc.c[2 * q].w, -kc.c[k1].w);
            }
            st = launch_dp_batch(NM, v, items_p, nitems, book_p, counters_p + (i - 2), hist, L, i - 2, has_next,
                                 /*has_prev=*/i - 1 >= 2, kc, Us, ((int64_t)i * nn - n_lo) * NM, p, tl.caps, ls,
                                 /*pdl_ok=*/true);
            count_launch(K_DP);
        }
        dp_timer.reset();
        if (st != HGM_OK) break;
        if ((e = cudaGetLastError()) != cudaSuccess) {
            st = cuda_fail(e, "K-DP launch");
            break;
        }
        {
            HostPhase hp_bt(HP_BT);
            Timer tm(ls, K_BT);
            st = v0 ? launch_backtrack_v0(v, di, ninst, hist, L, bt, p, ls)
                    : launch_backtrack_warp(v, di, ninst, hist, L, bt, p, ls);
            count_launch(K_BT);
        }
        if (st == HGM_OK && (e = cudaGetLastError()) != cudaSuccess) st = cuda_fail(e, "K-BT launch");
    }
    if (nlanes == 2) {  // join: the caller's stream waits for the second lane
        cudaEventRecord(ev_join, lanes[1].s);
        cudaStreamWaitEvent(s, ev_join, 0);
        cudaEventDestroy(ev_fork);
        cudaEventDestroy(ev_join);
    }
    cudaEventRecord(scr.done, s);  // the next user of the scratch buffers waits for this call's kernels
    return st;
}

}  // namespace hgm
