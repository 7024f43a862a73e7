// scene.cu -- scene index build and model chain build (a1).
//
// Scene (§3.4): stable sort of the points by frame, the
// minnode table first_tab[f] = first node with frame >= f (R4), and the pair
// band: for every node a, its successors c in frames (t'(a), t'(a) + T_max),
// which are the contiguous node range [minnode(t'(a)+1), minnode(t'(a)+T_max)).
// The band stores the ray direction theta(a->c) (K-G) and a coincidence flag; the
// padded copy K-DP stages (theta_pad) holds NaN instead of the direction of a
// zero-length ray, so the flag travels with the angle.
// Every admissible DP state (b, a) is one band entry, and every
// per-candidate operand of the recursion is a band entry too.
//
// Model (§2.1): one most-salient point per occupied frame,
// ordered by frame, plus per-triple constants of Eqs. 4-6 (gaps, model angles).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>

#include "hgm_device.cuh"
#include "hgm_internal.cuh"

namespace hgm {

__global__ void k_iota(int32_t *v, int64_t n) {
    int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k < n) v[k] = (int32_t)k;
}

// gather the sorted nodes; descriptors padded to Fp with zeros
// gather the sorted nodes; descriptors padded to Fp with zeros; *bad |= 1 on a
// non-finite coordinate or descriptor component (rejected by the caller: a NaN
// position would read as a coincidence flag in K-DP)
__global__ void k_gather(int64_t n, int F, int Fp, const int32_t *__restrict__ order, const int32_t *__restrict__ tk,
                         const float *__restrict__ x, const float *__restrict__ y, const float *__restrict__ feat,
                         const int64_t *__restrict__ id, int32_t *ot, float *ox, float *oy, float *of, int64_t *oid,
                         int *bad) {
    int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= n) return;
    int32_t src = order[k];
    ot[k] = tk[k];
    const float px = x[src], py = y[src];
    ox[k] = px;
    oy[k] = py;
    if (oid) oid[k] = id ? id[src] : (int64_t)src;
    const float *fr = feat + (int64_t)src * F;
    float *fo = of + k * (int64_t)Fp;
    bool ok = isfinite(px) && isfinite(py);
    for (int j = 0; j < Fp; ++j) {
        const float v = j < F ? fr[j] : 0.0f;
        ok = ok && isfinite(v);
        fo[j] = v;
    }
    if (!ok) atomicOr(bad, 1);
}

// *bad |= 1 if a model point has a non-finite coordinate, saliency or descriptor component
__global__ void k_check_finite(int64_t n, int F, const float *__restrict__ x, const float *__restrict__ y,
                               const float *__restrict__ sal, const float *__restrict__ feat, int *bad) {
    bool ok = true;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n * (int64_t)F;
         k += (int64_t)gridDim.x * blockDim.x) {
        ok = ok && isfinite(feat[k]);
        if (k < n) ok = ok && isfinite(x[k]) && isfinite(y[k]) && isfinite(sal[k]);  // sal never NULL here
    }
    if (!ok) atomicOr(bad, 1);
}

// first_tab[f] = minnode(f) for f in [0, fmax+1]; each f is written once
__global__ void k_first_tab(int64_t S, const int32_t *__restrict__ t, int32_t *first_tab) {
    int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (n > S) return;
    if (n == S) {
        first_tab[t[S - 1] + 1] = (int32_t)S;
        return;
    }
    int lo = n == 0 ? 0 : t[n - 1] + 1;
    for (int f = lo; f <= t[n]; ++f) first_tab[f] = (int32_t)n;
}

__global__ void k_rowlen(int64_t S, int T_max, int fmax, const int32_t *__restrict__ t,
                         const int32_t *__restrict__ ft, int32_t *rowlen) {
    int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (a > S) return;
    if (a == S) {
        rowlen[S] = 0;
        return;
    }
    int lo = first_at(ft, fmax, (int)S, t[a] + 1);
    int hi = first_at(ft, fmax, (int)S, t[a] + T_max);
    rowlen[a] = hi - lo;
}

__global__ void k_padlen(int64_t S, const int32_t *__restrict__ rowlen, int32_t *padlen) {
    int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (a > S) return;
    // padded length = 1 (mod 4): consecutive rows start in distinct 32-byte bank groups of
    // K-DP's candidate entries (and on distinct 4-byte banks of its direction rows)
    padlen[a] = a == S ? 0 : rowlen[a] + ((5 - (rowlen[a] & 3)) & 3);
}

// K-G: direction band theta(a->c) and coincidence flags, one thread per row a
__global__ void k_band(int64_t S, int T_max, int fmax, const int32_t *__restrict__ t, const float *__restrict__ x,
                       const float *__restrict__ y, const int32_t *__restrict__ ft, const int32_t *__restrict__ qstart,
                       const int32_t *__restrict__ qpad, float *theta, float *theta_pad, uint8_t *coinc,
                       uint16_t *cpre, int32_t *prow, int32_t *prow_pad, int32_t *rfc, int32_t *rlc) {
    int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (a >= S) return;
    int lo = first_at(ft, fmax, (int)S, t[a] + 1);
    int hi = first_at(ft, fmax, (int)S, t[a] + T_max);
    float ax = x[a], ay = y[a];
    int64_t p = qstart[a];
    float *tp = theta_pad + qpad[a];
    int32_t *rp = prow_pad + qpad[a];
    unsigned run = 0;
    int fc = 0x7fffffff, lc = -1;
    for (int c = lo; c < hi; ++c, ++p) {
        float cx = x[c], cy = y[c];
        const bool co = ax == cx && ay == cy;
        const float th = dir_of(ax, ay, cx, cy);
        theta[p] = th;
        tp[c - lo] = co ? __int_as_float(0x7fc00000) : th;  // K-DP's copy: NaN marks a zero-length ray (R10)
        rp[c - lo] = (int32_t)a;
        coinc[p] = co ? 1 : 0;
        run += co ? 1u : 0u;
        cpre[p] = (uint16_t)min(run, 65535u);
        prow[p] = (int32_t)a;
        if (co) {
            fc = min(fc, c - lo);
            lc = c - lo;
        }
    }
    for (int q = hi - lo; q < qpad[a + 1] - qpad[a]; ++q) {  // padding slots
        tp[q] = 0.f;
        rp[q] = -1;
    }
    rfc[a] = fc;
    rlc[a] = lc;
}

__global__ void k_ninfo(int64_t S, int fmax, const int32_t *__restrict__ t, const int32_t *__restrict__ ft,
                        const int32_t *__restrict__ qstart, const int32_t *__restrict__ qpad, int4 *ninfo) {
    int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (a >= S) return;
    ninfo[a] = make_int4(t[a], first_at(ft, fmax, (int)S, t[a] + 1), qstart[a], qpad[a]);
}

static hgm_status sort_by_frame(const int32_t *frame, int64_t n, int32_t *keys_out, int32_t *order,
                                cudaStream_t s) {
    DevBuf iota, tmp;
    HGM_TRY(iota.alloc(sizeof(int32_t) * n, s));
    k_iota<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(iota.as<int32_t>(), n);
    size_t tmp_bytes = 0;
    HGM_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, frame, keys_out, iota.as<int32_t>(), order,
                                             (int)n, 0, 32, s));
    HGM_TRY(tmp.alloc(tmp_bytes, s));
    // radix sort is stable: equal frames keep input order
    HGM_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, frame, keys_out, iota.as<int32_t>(), order,
                                             (int)n, 0, 32, s));
    count_launch(K_SCENE, 2);
    return HGM_OK;
}

static void free_scene_dev(hgm_scene *sc) {
    void *ptrs[] = {sc->t,      sc->x,     sc->y,     sc->feat, sc->id,  sc->first_tab,
                    sc->qstart, sc->theta, sc->coinc, sc->cpre, sc->prow,
                    sc->qpad,   sc->theta_pad, sc->prow_pad, sc->rfc, sc->rlc, sc->ninfo};
    for (void *p : ptrs)
        if (p) cudaFree(p);
}

hgm_status scene_build_device(const hgm_points *pts, int32_t T_max, cudaStream_t s, hgm_scene **out) {
    const int64_t n = pts->n;
    if (n > (int64_t)INT32_MAX - 1) return fail(HGM_ERR_INVALID_ARGUMENT, "too many scene points");
    Timer tm(s, K_SCENE);
    hgm_scene *sc = new hgm_scene();
    HGM_CUDA(cudaGetDevice(&sc->device));
    sc->S = n;
    sc->F = pts->F;
    sc->Fp = pad4(pts->F);
    sc->T_max = T_max;
    auto dmalloc = [&](auto **ptr, size_t bytes) { return cudaMallocAsync((void **)ptr, bytes, s); };
    auto bail = [&](hgm_status st) {
        free_scene_dev(sc);
        delete sc;
        return st;
    };
#define SC_CUDA(call)                                                    \
    do {                                                                 \
        cudaError_t e__ = (call);                                        \
        if (e__ != cudaSuccess) return bail(cuda_fail(e__, #call));      \
    } while (0)
    SC_CUDA(dmalloc(&sc->t, sizeof(int32_t) * (n + 4)));  // + 16 B slack on arrays K-DP bulk-copies
    SC_CUDA(dmalloc(&sc->x, sizeof(float) * n));
    SC_CUDA(dmalloc(&sc->y, sizeof(float) * n));
    SC_CUDA(dmalloc(&sc->feat, sizeof(float) * n * sc->Fp));
    SC_CUDA(dmalloc(&sc->id, sizeof(int64_t) * n));
    SC_CUDA(dmalloc(&sc->qstart, sizeof(int32_t) * (n + 1)));
    DevBuf badbuf;
    if (badbuf.alloc(sizeof(int), s) != HGM_OK) return bail(HGM_ERR_OUT_OF_MEMORY);
    SC_CUDA(cudaMemsetAsync(badbuf.p, 0, sizeof(int), s));
    {
        DevBuf order;
        if (order.alloc(sizeof(int32_t) * n, s) != HGM_OK) return bail(HGM_ERR_OUT_OF_MEMORY);
        hgm_status st = sort_by_frame(pts->frame, n, sc->t, order.as<int32_t>(), s);
        if (st != HGM_OK) return bail(st);
        unsigned g = (unsigned)((n + 255) / 256);
        k_gather<<<g, 256, 0, s>>>(n, pts->F, sc->Fp, order.as<int32_t>(), sc->t, pts->x, pts->y, pts->feat, pts->id,
                                   sc->t, sc->x, sc->y, sc->feat, sc->id, badbuf.as<int>());
        count_launch(K_SCENE);
        SC_CUDA(cudaGetLastError());
    }
    int32_t tt[3];
    SC_CUDA(cudaMemcpyAsync(&tt[0], sc->t, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    SC_CUDA(cudaMemcpyAsync(&tt[1], sc->t + n - 1, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    SC_CUDA(cudaMemcpyAsync(&tt[2], badbuf.p, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    SC_CUDA(cudaStreamSynchronize(s));
    if (tt[0] < 0) return bail(fail(HGM_ERR_INVALID_ARGUMENT, "negative frame index"));
    if (tt[1] > HGM_MAX_FRAME) return bail(fail(HGM_ERR_INVALID_ARGUMENT, "frame index above 2^26 (frames must be a video's frame numbers)"));
    if (tt[2]) return bail(fail(HGM_ERR_INVALID_ARGUMENT, "non-finite coordinate or descriptor component"));
    sc->fmax = tt[1];
    // T_max at or above the scene's frame span + 1 admits every pair: the band is built for
    // min(T_max, fmax + 1), identical in result and free of int overflow in t + T
    const int Tb = (int)std::min<int64_t>(T_max, (int64_t)sc->fmax + 1);
    SC_CUDA(dmalloc(&sc->first_tab, sizeof(int32_t) * (sc->fmax + 2 + 4)));
    k_first_tab<<<(unsigned)((n + 1 + 255) / 256), 256, 0, s>>>(n, sc->t, sc->first_tab);
    DevBuf rowlen, tmp;
    if (rowlen.alloc(sizeof(int32_t) * (n + 1), s) != HGM_OK) return bail(HGM_ERR_OUT_OF_MEMORY);
    k_rowlen<<<(unsigned)((n + 1 + 255) / 256), 256, 0, s>>>(n, Tb, sc->fmax, sc->t, sc->first_tab,
                                                             rowlen.as<int32_t>());
    count_launch(K_SCENE, 2);
    size_t tb = 0;
    SC_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, rowlen.as<int32_t>(), sc->qstart, (int)(n + 1), s));
    if (tmp.alloc(tb, s) != HGM_OK) return bail(HGM_ERR_OUT_OF_MEMORY);
    SC_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, rowlen.as<int32_t>(), sc->qstart, (int)(n + 1), s));
    // padded band offsets (odd row lengths)
    SC_CUDA(dmalloc(&sc->qpad, sizeof(int32_t) * (n + 1)));
    {
        DevBuf padlen;
        if (padlen.alloc(sizeof(int32_t) * (n + 1), s) != HGM_OK) return bail(HGM_ERR_OUT_OF_MEMORY);
        k_padlen<<<(unsigned)((n + 1 + 255) / 256), 256, 0, s>>>(n, rowlen.as<int32_t>(), padlen.as<int32_t>());
        SC_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, padlen.as<int32_t>(), sc->qpad, (int)(n + 1), s));
    }
    count_launch(K_SCENE, 3);
    sc->first_h.resize(sc->fmax + 2);
    sc->qstart_h.resize(n + 1);
    sc->qpad_h.resize(n + 1);
    SC_CUDA(cudaMemcpyAsync(sc->first_h.data(), sc->first_tab, sizeof(int32_t) * (sc->fmax + 2),
                            cudaMemcpyDeviceToHost, s));
    SC_CUDA(cudaMemcpyAsync(sc->qstart_h.data(), sc->qstart, sizeof(int32_t) * (n + 1), cudaMemcpyDeviceToHost, s));
    SC_CUDA(cudaMemcpyAsync(sc->qpad_h.data(), sc->qpad, sizeof(int32_t) * (n + 1), cudaMemcpyDeviceToHost, s));
    SC_CUDA(cudaStreamSynchronize(s));
    sc->npairs = sc->qstart_h[n];
    if (sc->qpad_h[n] < sc->npairs) return bail(fail(HGM_ERR_INVALID_ARGUMENT, "pair band exceeds 2^31 entries"));
    SC_CUDA(dmalloc(&sc->rfc, sizeof(int32_t) * (n + 4)));
    SC_CUDA(dmalloc(&sc->rlc, sizeof(int32_t) * (n + 4)));
    SC_CUDA(dmalloc(&sc->theta_pad, sizeof(float) * ((int64_t)sc->qpad_h[n] + 4)));
    SC_CUDA(dmalloc(&sc->prow_pad, sizeof(int32_t) * ((int64_t)sc->qpad_h[n] + 4)));
    if (sc->npairs > 0) {
        SC_CUDA(dmalloc(&sc->theta, sizeof(float) * sc->npairs));
        SC_CUDA(dmalloc(&sc->coinc, sizeof(uint8_t) * sc->npairs));
        SC_CUDA(dmalloc(&sc->cpre, sizeof(uint16_t) * sc->npairs));
        SC_CUDA(dmalloc(&sc->prow, sizeof(int32_t) * sc->npairs));
    }
    k_band<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(n, Tb, sc->fmax, sc->t, sc->x, sc->y, sc->first_tab,
                                                       sc->qstart, sc->qpad, sc->theta, sc->theta_pad, sc->coinc,
                                                       sc->cpre, sc->prow, sc->prow_pad, sc->rfc, sc->rlc);
    SC_CUDA(dmalloc(&sc->ninfo, sizeof(int4) * n));
    k_ninfo<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, sc->fmax, sc->t, sc->first_tab, sc->qstart, sc->qpad,
                                                        sc->ninfo);
    count_launch(K_SCENE, 2);
    SC_CUDA(cudaGetLastError());
    SC_CUDA(cudaStreamSynchronize(s));
#undef SC_CUDA
    *out = sc;
    return HGM_OK;
}

// ------------------------------------------------------------------ model
// After the stable sort, the first point of each frame run is the earliest
// input point of that frame; the max-saliency scan with a strict ">" keeps the
// earliest one on ties (R-D1).
__global__ void k_model_select(int64_t n, const int32_t *__restrict__ t, const int32_t *__restrict__ order,
                               const float *__restrict__ sal, int rank, int32_t *sel, int32_t *M_out) {
    // one thread: n is a model's point count (hundreds).  Per frame, the point of
    // saliency rank `rank` (0 = most salient; rank r = chain r of the
    // independent-chains model); ties: earlier input point first
    // (the frame sort is stable, so group position = input order).
    if (threadIdx.x == 0) {
        int m = 0;
        for (int64_t k = 0; k < n;) {
            int64_t j = k + 1;
            while (j < n && t[j] == t[k]) ++j;
            for (int64_t q = k; q < j; ++q) {
                int beaten = 0;
                const float sq = sal[order[q]];
                for (int64_t r = k; r < j; ++r) {
                    const float sr = sal[order[r]];
                    beaten += (sr > sq || (sr == sq && r < q)) ? 1 : 0;
                }
                if (beaten == rank) sel[m++] = (int32_t)q;
            }
            k = j;
        }
        *M_out = m;
    }
}

__global__ void k_model_gather(int M, int F, int Fp, const int32_t *__restrict__ sel, const int32_t *__restrict__ t,
                               const int32_t *__restrict__ order, const float *__restrict__ x,
                               const float *__restrict__ y, const float *__restrict__ feat, int32_t *ot, float *ox,
                               float *oy, float *of) {
    int i = blockIdx.x;
    if (i >= M) return;
    int k = sel[i];
    int src = order[k];
    if (threadIdx.x == 0) {
        ot[i] = t[k];
        ox[i] = x[src];
        oy[i] = y[src];
    }
    for (int j = threadIdx.x; j < Fp; j += blockDim.x) of[(int64_t)i * Fp + j] = j < F ? feat[(int64_t)src * F + j] : 0.f;
}

// Per-triple model constants for steps i >= 2 (0-based): gaps of Eq. 5 and the
// model angles of Eq. 6 in the fold representation of hgm_device.cuh.
__global__ void k_model_steps(int M, const int32_t *__restrict__ t, const float *__restrict__ x,
                              const float *__restrict__ y, float4 *step) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= M) return;
    if (i < 2) {
        step[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        return;
    }
    int a = i - 2, b = i - 1, c = i;
    float th_ab = dir_of(x[a], y[a], x[b], y[b]);
    float th_bc = dir_of(x[b], y[b], x[c], y[c]);
    float th_ac = dir_of(x[a], y[a], x[c], y[c]);
    bool co_ab = x[a] == x[b] && y[a] == y[b];
    bool co_bc = x[b] == x[c] && y[b] == y[c];
    bool co_ac = x[a] == x[c] && y[a] == y[c];
    float A1 = (co_bc || co_ab) ? 0.0f : fold(th_bc, th_ab);      // model angle at i-1
    float K2 = (co_bc || co_ac) ? HGM_PI_F : fold(th_bc, th_ac);  // pi - model angle at i
    step[i] = make_float4((float)(t[c] - t[b]), (float)(t[b] - t[a]), A1, K2);
}

hgm_status model_build_device(const hgm_points *pts, int rank, cudaStream_t s, hgm_model **out) {
    const int64_t n = pts->n;
    if (n > 1000000) return fail(HGM_ERR_INVALID_ARGUMENT, "model point set too large");
    Timer tm(s, K_MODEL);
    DevBuf keys, order, sel, Mdev;
    HGM_TRY(keys.alloc(sizeof(int32_t) * n, s));
    HGM_TRY(order.alloc(sizeof(int32_t) * n, s));
    HGM_TRY(sel.alloc(sizeof(int32_t) * n, s));
    HGM_TRY(Mdev.alloc(sizeof(int32_t), s));
    DevBuf bad, zsal;
    const float *sal = pts->saliency;
    if (!sal) {  // no detector confidence given: all points equally salient (earliest wins, R-D1)
        HGM_TRY(zsal.alloc(sizeof(float) * n, s));
        HGM_CUDA(cudaMemsetAsync(zsal.p, 0, sizeof(float) * n, s));
        sal = zsal.as<float>();
    }
    HGM_TRY(bad.alloc(sizeof(int), s));
    HGM_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), s));
    k_check_finite<<<(unsigned)std::min<int64_t>((n * pts->F + 255) / 256, 1024), 256, 0, s>>>(
        n, pts->F, pts->x, pts->y, sal, pts->feat, bad.as<int>());
    HGM_TRY(sort_by_frame(pts->frame, n, keys.as<int32_t>(), order.as<int32_t>(), s));
    k_model_select<<<1, 32, 0, s>>>(n, keys.as<int32_t>(), order.as<int32_t>(), sal, rank,
                                    sel.as<int32_t>(), Mdev.as<int32_t>());
    count_launch(K_MODEL);
    int32_t M = 0, t0 = 0, t1 = 0, nbad = 0;
    HGM_CUDA(cudaMemcpyAsync(&M, Mdev.p, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    HGM_CUDA(cudaMemcpyAsync(&t0, keys.p, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    HGM_CUDA(cudaMemcpyAsync(&t1, keys.as<int32_t>() + n - 1, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    HGM_CUDA(cudaMemcpyAsync(&nbad, bad.p, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    HGM_CUDA(cudaStreamSynchronize(s));
    if (t0 < 0) return fail(HGM_ERR_INVALID_ARGUMENT, "negative frame index");
    if (t1 > HGM_MAX_FRAME) return fail(HGM_ERR_INVALID_ARGUMENT, "frame index above 2^26");
    if (nbad) return fail(HGM_ERR_INVALID_ARGUMENT, "non-finite coordinate, saliency or descriptor component");
    if (M == 0) return fail(HGM_ERR_EMPTY_POINT_SET, "no frame has a point of this saliency rank");
    hgm_model *m = new hgm_model();
    HGM_CUDA(cudaGetDevice(&m->device));
    m->M = M;
    m->F = pts->F;
    m->Fp = pad4(pts->F);
    auto dmalloc = [&](auto **ptr, size_t bytes) { return cudaMallocAsync((void **)ptr, bytes, s); };
    cudaError_t e = cudaSuccess;
    if (e == cudaSuccess) e = dmalloc(&m->t, sizeof(int32_t) * M);
    if (e == cudaSuccess) e = dmalloc(&m->x, sizeof(float) * M);
    if (e == cudaSuccess) e = dmalloc(&m->y, sizeof(float) * M);
    if (e == cudaSuccess) e = dmalloc(&m->feat, sizeof(float) * M * m->Fp);
    if (e == cudaSuccess) e = dmalloc(&m->step, sizeof(float4) * M);
    if (e != cudaSuccess) {
        hgm_free_model(m);
        return cuda_fail(e, "cudaMalloc(model)");
    }
    k_model_gather<<<M, 64, 0, s>>>(M, pts->F, m->Fp, sel.as<int32_t>(), keys.as<int32_t>(), order.as<int32_t>(),
                                    pts->x, pts->y, pts->feat, m->t, m->x, m->y, m->feat);
    k_model_steps<<<(M + 63) / 64, 64, 0, s>>>(M, m->t, m->x, m->y, m->step);
    count_launch(K_MODEL, 2);
    m->t_h.resize(M);
    m->step_h.resize(M);
    HGM_CUDA(cudaMemcpyAsync(m->t_h.data(), m->t, sizeof(int32_t) * M, cudaMemcpyDeviceToHost, s));
    HGM_CUDA(cudaMemcpyAsync(m->step_h.data(), m->step, sizeof(float4) * M, cudaMemcpyDeviceToHost, s));
    HGM_CUDA(cudaStreamSynchronize(s));
    *out = m;
    return HGM_OK;
}

}  // namespace hgm
