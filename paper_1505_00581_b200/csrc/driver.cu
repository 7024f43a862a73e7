// driver.cu -- host orchestration of one model batch at every offset:
// window descriptors, tile geometry, chunking of the alpha history, one K-DP
// launch per recursion step i = M..3 (Eq. 10, the paper's host loop of
// Alg. 2 with the whole batch of windows per launch), then K-BT.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "dp_common.cuh"

namespace hgm {

hgm_status launch_dp_batch(int NM, const SceneView &v, const InstDesc *dinst, int ninst, float *hist, int64_t L,
                           int layer, bool has_next, bool has_prev, const StepConstB &kc, const float *msg,
                           const DPParams &p, const TileGeom &tg, cudaStream_t s);
hgm_status launch_msg(int NM, const SceneView &v, const InstDesc *dinst, int ninst, int max_np, int max_sw,
                      float *hist, int64_t L, int layer, bool has_next, bool init, const StepConstB &kc,
                      const float *Ui, float *msg, const DPParams &p, int W, cudaStream_t s);
size_t dp_batch_smem(const TileGeom &tg, int T, int NM);
hgm_status launch_backtrack_warp(const SceneView &v, const InstDesc *dinst, int ninst, const float *hist, int64_t L,
                                 const BTArgs &bt, const DPParams &p, cudaStream_t s);
hgm_status launch_dp_v0(const SceneView &v, const InstDesc *dinst, int ninst, int64_t maxNs, float *hist, int64_t L,
                        int layer, bool has_next, const StepConst &kc, const float *U, int64_t n_lo, const DPParams &p,
                        cudaStream_t s);
hgm_status launch_backtrack_v0(const SceneView &v, const InstDesc *dinst, int ninst, const float *hist, int64_t L,
                               const BTArgs &bt, const DPParams &p, cudaStream_t s);

static inline int host_first(const hgm_scene *sc, int64_t f) {
    if (f <= 0) return 0;
    if (f > sc->fmax) return (int)sc->S;
    return sc->first_h[f];
}

// second stream of the chunk pipeline, one per device
static cudaStream_t aux_stream(int device) {
    static std::mutex mu;
    static cudaStream_t as[64] = {};
    std::lock_guard<std::mutex> lk(mu);
    if (device < 0 || device >= 64) return nullptr;
    if (!as[device]) cudaStreamCreateWithFlags(&as[device], cudaStreamNonBlocking);
    return as[device];
}

bool use_v0_kernels() {
    const char *e = getenv("HGM_KERNEL");
    return e && strcmp(e, "v0") == 0;
}

// Shared-memory capacities of a K-DP tile of FT b-frames, as upper bounds over
// every tile start the call can produce (host, from the frame index); the
// largest FT within the budget wins.
static bool tile_geometry(const hgm_scene *sc, const hgm_offsets &o, int T, int NM, TileGeom *tg) {
    const int64_t f_lo = (int64_t)o.first_frame - T - 1;
    const int64_t f_hi = (int64_t)o.first_frame + (int64_t)(o.count - 1) * o.stride + o.window + T + 1;
    auto Q = [&](int n) { return (int64_t)sc->qstart_h[n]; };
    auto QP = [&](int n) { return (int64_t)sc->qpad_h[n]; };
    static const int cand[] = {8, 6, 5, 4, 3, 2, 1};
    const char *env = getenv("HGM_TILE_FRAMES");
    const int want = env ? atoi(env) : 0;
    for (int pass = 0; pass < 2; ++pass) {
        for (int FT : cand) {
            if (want > 0 && FT != want) continue;
            if (FT * (T - 1) > 255) continue;  // segment ids are bytes
            TileGeom g{};
            g.FT = FT;
            g.W = o.window;
            g.ntile = (o.window + FT - 1) / FT;
            int64_t NB = 1, NA = 1, TH = 1, MT = 1, NST = 1;
            for (int64_t F0 = f_lo; F0 <= f_hi; ++F0) {
                const int B0 = host_first(sc, F0), B1 = host_first(sc, F0 + FT), A0 = host_first(sc, F0 - T + 1);
                NB = std::max<int64_t>(NB, B1 - B0);
                NA = std::max<int64_t>(NA, B1 - A0);
                TH = std::max<int64_t>(TH, QP(B1) - QP(A0) + 8);  // one aligned copy of the padded rows
                MT = std::max<int64_t>(MT, QP(B1) - QP(B0) + 8);  // message rows, padded, + alignment slack
                int64_t nst = 0;
                for (int64_t f = F0; f < F0 + FT; ++f)
                    nst += (int64_t)(host_first(sc, f + 1) - host_first(sc, f)) *
                           (host_first(sc, f) - host_first(sc, f - T + 1));
                NST = std::max(NST, nst);
            }
            g.NB = (int)NB;
            g.NA = (int)NA;
            g.TH = (int)TH;
            g.MT = (int)MT;
            g.NST = (int)NST;
            const size_t budget = pass == 0 ? 60 * 1024 : 200 * 1024;
            if (dp_batch_smem(g, T, NM) <= budget) {
                *tg = g;
                return true;
            }
        }
    }
    return false;
}

// Match NM models of equal chain length M at every offset.
// U: batched unary table U[((i * nn) + (n - n_lo)) * NM + k].
hgm_status match_batch(const hgm_model *const *models, int NM, const hgm_scene *sc, const hgm_params &pp,
                       const hgm_offsets &o, const float *U, int64_t n_lo, int64_t nn, const MatchOut *outs,
                       cudaStream_t s) {
    const int count = o.count, M = models[0]->M;
    if (count <= 0) return HGM_OK;
    if (NM < 1 || NM > MAX_BATCH) return fail(HGM_ERR_INVALID_ARGUMENT, "model batch size must be 1..8");
    const bool v0 = use_v0_kernels();
    if (v0 && NM != 1) return fail(HGM_ERR_INVALID_ARGUMENT, "v0 kernels take one model at a time");
    std::vector<InstDesc> all(count);
    for (int k = 0; k < count; ++k) {
        const int64_t of = (int64_t)o.first_frame + (int64_t)k * o.stride;
        InstDesc d{};
        d.wb = host_first(sc, of);
        d.we = host_first(sc, of + o.window);
        d.pbase = sc->qstart_h[d.wb];
        d.np = sc->qstart_h[d.we] - sc->qstart_h[d.wb];
        d.out = k;
        d.o = (int32_t)of;
        all[k] = d;
    }
    TileGeom tg{};
    if (!v0 && !tile_geometry(sc, o, pp.T, NM, &tg))
        return fail(HGM_ERR_INVALID_ARGUMENT, "window too dense for the shared-memory tile (reduce T or window)");
    DPParams p;
    p.l1 = pp.lambda1;
    p.l2 = pp.lambda2;
    p.l23 = pp.lambda2 * pp.lambda3;  // one IEEE single multiply
    p.W = pp.w_dummy;
    p.l1W = pp.lambda1 * pp.w_dummy;
    p.T = pp.T;
    const SceneView v{sc->t,    sc->first_tab, sc->qstart, sc->theta,     sc->coinc, sc->cpre,
                      sc->prow, sc->id,        sc->qpad,   sc->theta_pad, sc->rfc,   sc->rlc,
                      sc->ninfo, sc->fmax,     (int)sc->S};
    const int nsteps = M >= 3 ? M - 2 : 0;
    // Windows are processed in chunks (the alpha history of a chunk must fit the
    // budget).  Chunks alternate between two streams, so the streaming K-MSG of
    // one chunk overlaps the compute-bound K-DP of the other on the same SMs.
    const int64_t budget_floats = (int64_t)3 << 29;  // alpha history per chunk: 6 GiB
    BTArgs bt{};
    bt.U = U;
    bt.nn = nn;
    bt.n_lo = n_lo;
    bt.NM = NM;
    bt.M = M;
    for (int k = 0; k < NM; ++k) {
        bt.step[k] = models[k]->step;
        bt.E[k] = outs[k].E;
        bt.A[k] = outs[k].A;
        bt.z[k] = outs[k].z;
    }
    const int NMP = nm_pad(NM);
    const char *cenv = getenv("HGM_CHUNK");  // windows per chunk (tuning knob)
    const int chunk_max = std::min(65535, cenv && atoi(cenv) > 0 ? atoi(cenv) : 4096);
    const char *senv = getenv("HGM_STREAMS");  // 2: alternate chunks over two streams (measured slower)
    const int nlanes = (senv && atoi(senv) == 2) ? 2 : 1;
    struct Lane {
        cudaStream_t s = nullptr;
        DevBuf hist, msg, dinst;
        int64_t hist_cap = 0, msg_cap = 0, dinst_cap = 0;
    } lanes[2];
    lanes[0].s = s;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    if (nlanes == 2) {
        lanes[1].s = aux_stream(sc->device);
        HGM_CUDA(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
        HGM_CUDA(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
        HGM_CUDA(cudaEventRecord(ev_fork, s));
        HGM_CUDA(cudaStreamWaitEvent(lanes[1].s, ev_fork, 0));
    }
    hgm_status st = HGM_OK;
    int chunk = 0;
    for (int k0 = 0; k0 < count && st == HGM_OK; ++chunk) {
        Lane &ln = lanes[chunk % nlanes];
        const cudaStream_t ls = ln.s;
        int64_t L = 0, maxNs = 1, MS = 0;
        int k1 = k0, max_sw = 1, max_np = 1;
        while (k1 < count && k1 - k0 < chunk_max) {
            InstDesc &d = all[k1];
            const int64_t ns = (int64_t)d.np + 2 * (int64_t)(d.we - d.wb) + 1;
            if (k1 > k0 && (L + ns * NM) * std::max(nsteps, 1) > budget_floats) break;
            d.off = L;
            L += ns * NM;
            d.ppad = sc->qpad_h[d.wb];
            d.moff = MS;
            MS += (((int64_t)sc->qpad_h[d.we] - d.ppad) * NMP + 3) & ~(int64_t)3;  // 16-byte aligned rows
            maxNs = std::max(maxNs, ns);
            max_sw = std::max(max_sw, d.we - d.wb);
            max_np = std::max(max_np, d.np);
            ++k1;
        }
        const int ninst = k1 - k0;
        if (ninst > ln.dinst_cap) {
            if ((st = ln.dinst.alloc(sizeof(InstDesc) * ninst, ls)) != HGM_OK) break;
            ln.dinst_cap = ninst;
        }
        cudaError_t e = cudaMemcpyAsync(ln.dinst.p, all.data() + k0, sizeof(InstDesc) * ninst,
                                        cudaMemcpyHostToDevice, ls);
        if (e != cudaSuccess) {
            st = cuda_fail(e, "cudaMemcpyAsync(instances)");
            break;
        }
        const int64_t need = L * nsteps;
        if (need > ln.hist_cap) {
            if ((st = ln.hist.alloc(sizeof(float) * need, ls)) != HGM_OK) break;
            ln.hist_cap = need;
        }
        if (!v0 && nsteps > 0 && MS + 4 > ln.msg_cap) {
            if ((st = ln.msg.alloc(sizeof(float) * (MS + 4), ls)) != HGM_OK) break;
            ln.msg_cap = MS + 4;
        }
        const InstDesc *di = ln.dinst.as<InstDesc>();
        float *hist = ln.hist.as<float>();
        auto Urow = [&](int i) { return U + ((int64_t)i * nn - n_lo) * NM; };  // batched row, Urow(i)[c*NM + k]
        for (int i = M - 1; i >= 2 && st == HGM_OK; --i) {
            const bool has_next = i + 1 <= M - 1;
            if (v0) {
                Timer tm(ls, K_DP);
                const float4 h = models[0]->step_h[i];
                const StepConst kc{h.x, h.y, h.z, h.w};
                st = launch_dp_v0(v, di, ninst, maxNs, hist, L, i - 2, has_next, kc, U + (int64_t)i * nn, n_lo, p, ls);
                count_launch(K_DP);
                continue;
            }
            StepConstB kc{};
            for (int k = 0; k < NM; ++k) kc.c[k] = models[k]->step_h[i];
            {
                Timer tm(ls, K_MSG);
                st = launch_msg(NM, v, di, ninst, max_np, max_sw, hist, L, i - 2, has_next, /*init=*/!has_next, kc,
                                Urow(i), ln.msg.as<float>(), p, o.window, ls);
                count_launch(K_MSG, has_next ? 1 : 2);
            }
            if (st != HGM_OK) break;
            {
                Timer tm(ls, K_DP);
                st = launch_dp_batch(NM, v, di, ninst, hist, L, i - 2, has_next, /*has_prev=*/i - 1 >= 2, kc,
                                     ln.msg.as<float>(), p, tg, ls);
                count_launch(K_DP);
            }
        }
        if (st != HGM_OK) break;
        if ((e = cudaGetLastError()) != cudaSuccess) {
            st = cuda_fail(e, "K-DP launch");
            break;
        }
        {
            Timer tm(ls, K_BT);
            st = v0 ? launch_backtrack_v0(v, di, ninst, hist, L, bt, p, ls)
                    : launch_backtrack_warp(v, di, ninst, hist, L, bt, p, ls);
            count_launch(K_BT);
        }
        if (st == HGM_OK && (e = cudaGetLastError()) != cudaSuccess) st = cuda_fail(e, "K-BT launch");
        k0 = k1;  // a lane's buffers are reused by its next chunk: stream order protects them
    }
    if (nlanes == 2) {  // join: the caller's stream waits for the second lane
        cudaEventRecord(ev_join, lanes[1].s);
        cudaStreamWaitEvent(s, ev_join, 0);
        cudaEventDestroy(ev_fork);
        cudaEventDestroy(ev_join);
    }
    return st;
}

}  // namespace hgm
