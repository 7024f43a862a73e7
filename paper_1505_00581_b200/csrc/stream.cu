// Streaming detection ("If the scene video is cut
// into smaller blocks of 60 frames, which is necessary for continuous video
// processing, real time performance can be achieved ... Additional processing will be
// required in order to treat overlapping blocks").
//
// Frames arrive in order.  After each push, every offset whose window [o, o + W) is
// complete (o + W <= frames pushed) and not yet reported is detected, exactly as a
// one-shot hgm_detect_actions over the whole stream would (same windows, same kernels):
// the stream keeps only the points of frames >= the next unreported offset o_next,
// rebases their frames to o_next - 1 (every quantity of the method depends on frame
// differences only), adds an anchor node at the rebased frame 0 (before every window),
// builds a scene index of them and runs the detect path on the completed offsets.
#include <algorithm>
#include <vector>

#include "hgm_internal.cuh"

struct hgm_stream {
    std::vector<const hgm_model *> models;
    hgm_params params{};
    int32_t window = 60, stride = 1, score_mode = 0, device = 0, F = 0;
    float threshold = 0.f;
    int64_t seen = 0;    // frames pushed so far
    int64_t o_next = 0;  // next unreported offset (a multiple of stride)
    // retained points (host), absolute frames >= o_next
    std::vector<int32_t> frame;
    std::vector<float> x, y, sal, feat;
};

using namespace hgm;

extern "C" {

hgm_status hgm_stream_create(const hgm_model *const *models, int32_t n_models, const hgm_params *params,
                             int32_t window, int32_t stride, int32_t score_mode, float threshold, int32_t device,
                             hgm_stream **out) {
    if (!out || !params) return fail(HGM_ERR_INVALID_ARGUMENT, "NULL argument");
    if (!models || n_models <= 0) return fail(HGM_ERR_EMPTY_POINT_SET, "empty model dictionary");
    if (window < 1 || stride < 1) return fail(HGM_ERR_INVALID_ARGUMENT, "window and stride must be >= 1");
    if (score_mode != 0 && score_mode != 1) return fail(HGM_ERR_INVALID_ARGUMENT, "score_mode must be 0 or 1");
    if (params->T < 1) return fail(HGM_ERR_INVALID_ARGUMENT, "T < 1");
    auto *st = new hgm_stream();
    for (int m = 0; m < n_models; ++m) {
        if (!models[m]) {
            delete st;
            return fail(HGM_ERR_INVALID_ARGUMENT, "NULL model handle");
        }
        st->models.push_back(models[m]);
    }
    st->F = models[0]->F;
    st->params = *params;
    st->window = window;
    st->stride = stride;
    st->score_mode = score_mode;
    st->threshold = threshold;
    st->device = device;
    *out = st;
    return HGM_OK;
}

hgm_status hgm_stream_push(hgm_stream *st, const hgm_points *pts, int32_t n_frames, int32_t capacity,
                           int32_t *winner, float *score, int32_t *n_out, int64_t *first_offset) {
    NvtxRange nvtx_("hgm_stream_push");
    if (!st || !n_out || !first_offset) return fail(HGM_ERR_INVALID_ARGUMENT, "NULL argument");
    if (n_frames < 0) return fail(HGM_ERR_INVALID_ARGUMENT, "n_frames < 0");
    *n_out = 0;
    *first_offset = st->o_next;
    // validate everything before the stream's state changes: a failed push leaves the
    // stream exactly as it was, so the caller can retry it (e.g. with more capacity)
    if (pts && pts->n > 0) {
        if (!pts->frame || !pts->x || !pts->y || !pts->feat) return fail(HGM_ERR_INVALID_ARGUMENT, "NULL point array");
        if (pts->F != st->F) return fail(HGM_ERR_DIMENSION_MISMATCH, "point and model descriptor lengths differ");
        for (int64_t k = 0; k < pts->n; ++k)
            if (pts->frame[k] < st->seen || pts->frame[k] >= st->seen + n_frames)
                return fail(HGM_ERR_INVALID_ARGUMENT, "pushed point outside the pushed frames [seen, seen + n_frames)");
    }
    const int64_t seen1 = st->seen + n_frames;
    const int64_t count = seen1 < st->o_next + st->window ? 0 : (seen1 - st->window - st->o_next) / st->stride + 1;
    if (count > INT32_MAX) return fail(HGM_ERR_INVALID_ARGUMENT, "too many offsets completed by one push");
    if (count > capacity || (count > 0 && (!winner || !score)))
        return fail(HGM_ERR_INVALID_ARGUMENT, "output capacity below the offsets this push completes");
    const size_t n_old = st->frame.size();
    auto rollback = [&](hgm_status stt) {
        st->frame.resize(n_old);
        st->x.resize(n_old);
        st->y.resize(n_old);
        st->sal.resize(n_old);
        st->feat.resize(n_old * (size_t)st->F);
        return stt;
    };
    if (pts && pts->n > 0) {
        for (int64_t k = 0; k < pts->n; ++k) {
            st->frame.push_back(pts->frame[k]);
            st->x.push_back(pts->x[k]);
            st->y.push_back(pts->y[k]);
            st->sal.push_back(pts->saliency ? pts->saliency[k] : 0.f);
        }
        st->feat.insert(st->feat.end(), pts->feat, pts->feat + pts->n * (int64_t)st->F);
    }
    if (count == 0) {
        st->seen = seen1;
        return HGM_OK;
    }
    // frames rebased to base = o_next - 1; an anchor node at rebased frame 0 lies before
    // every window [1 + k * stride, ...) so it is never a label (R13), and it keeps the
    // point set non-empty through silent stretches (windows without points are valid)
    const int64_t base = st->o_next - 1;
    const int64_t n = (int64_t)st->frame.size(), F = st->F;
    std::vector<int32_t> rf((size_t)n + 1);
    std::vector<float> rx((size_t)n + 1), ry((size_t)n + 1), rs((size_t)n + 1), rfeat((size_t)((n + 1) * F));
    rf[0] = 0;
    rx[0] = ry[0] = rs[0] = 0.f;
    std::fill(rfeat.begin(), rfeat.begin() + F, 0.f);
    for (int64_t k = 0; k < n; ++k) rf[(size_t)k + 1] = (int32_t)(st->frame[(size_t)k] - base);
    std::copy(st->x.begin(), st->x.end(), rx.begin() + 1);
    std::copy(st->y.begin(), st->y.end(), ry.begin() + 1);
    std::copy(st->sal.begin(), st->sal.end(), rs.begin() + 1);
    std::copy(st->feat.begin(), st->feat.end(), rfeat.begin() + F);
    hgm_points hp{n + 1, st->F, rf.data(), rx.data(), ry.data(), rs.data(), rfeat.data(), nullptr};
    hgm_scene *scene = nullptr;
    hgm_status bs = hgm_build_scene_index(&hp, st->device, st->params.T, &scene);
    if (bs != HGM_OK) return rollback(bs);
    hgm_offsets o{1, st->stride, (int32_t)count, st->window};
    const hgm_status ds = hgm_detect_actions(st->models.data(), (int32_t)st->models.size(), scene, &st->params, &o,
                                             st->score_mode, st->threshold, winner, score, nullptr, nullptr);
    hgm_free_scene(scene);
    if (ds != HGM_OK) return rollback(ds);
    const cudaError_t se = cudaStreamSynchronize(nullptr);
    if (se != cudaSuccess) return rollback(cuda_fail(se, "cudaStreamSynchronize(stream push)"));
    st->seen = seen1;
    *n_out = (int32_t)count;
    st->o_next += count * st->stride;
    // drop the points no later window reads (frames < o_next)
    int64_t w = 0;
    for (int64_t k = 0; k < n; ++k) {
        if (st->frame[(size_t)k] < st->o_next) continue;
        st->frame[(size_t)w] = st->frame[(size_t)k];
        st->x[(size_t)w] = st->x[(size_t)k];
        st->y[(size_t)w] = st->y[(size_t)k];
        st->sal[(size_t)w] = st->sal[(size_t)k];
        if (w != k)
            std::copy(st->feat.begin() + k * st->F, st->feat.begin() + (k + 1) * st->F, st->feat.begin() + w * st->F);
        ++w;
    }
    st->frame.resize((size_t)w);
    st->x.resize((size_t)w);
    st->y.resize((size_t)w);
    st->sal.resize((size_t)w);
    st->feat.resize((size_t)(w * st->F));
    return HGM_OK;
}

void hgm_stream_free(hgm_stream *st) { delete st; }

}  // extern "C"
