/*
 * hgm.h -- C ABI of libhgm.so: exact space-time hypergraph matching of a
 * second-order model chain against every temporal offset of a scene
 * (Lombardi, Wolf, Celiktutan, Sankur, arXiv 1505.00581), B200 (sm_100a).
 *
 * Citations: "P:Lnnn" = line of the paper source with its section /
 * equation; readings R1..R16 of silent or garbled passages are listed in
 * DESIGN.md §2 (same numbering as SURVEY.md §8(c) A1..A16).
 *
 * General conventions
 *  - Every entry point returns hgm_status; no C++ exception crosses the ABI.
 *    On a non-OK status, hgm_last_error() returns a thread-local message.
 *  - Input point arrays are BORROWED for the duration of the call and copied.
 *  - Handles (hgm_model, hgm_scene) are library-owned, immutable after build,
 *    safe for concurrent reads; release them with hgm_free_*.
 *  - Output buffers may be device pointers (written asynchronously on the
 *    caller's stream, stream-ordered) or host pointers (the call copies the
 *    results back and synchronises the stream before returning).
 *  - The library computes only on the GPU.  There is no CPU fallback: with no
 *    usable CUDA device every call returns HGM_ERR_CUDA.
 */
#ifndef HGM_H
#define HGM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    HGM_OK = 0,
    HGM_ERR_EMPTY_POINT_SET = 1,     /* n == 0 where points are required; n_models == 0 */
    HGM_ERR_DIMENSION_MISMATCH = 2,  /* descriptor length F differs between model(s) and scene */
    HGM_ERR_INVALID_ARGUMENT = 3,    /* NULL pointer, non-finite or negative lambda / W^d,
                                        T < 1, T > scene T_max, window < 1, stride < 1,
                                        count < 0, negative frame, frame > 2^26, offsets
                                        beyond +-2^26 frames, non-finite x / y / saliency /
                                        descriptor component, size overflow */
    HGM_ERR_OUT_OF_MEMORY = 4,       /* device allocation failed */
    HGM_ERR_CUDA = 5                 /* any other CUDA runtime error (incl. no device) */
} hgm_status;

typedef struct hgm_model hgm_model; /* opaque: model chain resident in HBM */
typedef struct hgm_scene hgm_scene; /* opaque: sorted scene + frame index + direction band */

/* One interest-point set (space-time position, detector
 * confidence and an F-dimensional appearance descriptor per point). */
typedef struct {
    int64_t n;              /* number of points */
    int32_t F;              /* descriptor length (162 for HoG/HoF) */
    const int32_t *frame;   /* [n] integer frame, 0 <= t <= 2^26 (a video's frame numbers) */
    const float *x, *y;     /* [n] pixel position */
    const float *saliency;  /* [n] detector confidence; used by the model builder only */
    const float *feat;      /* [n*F] row-major descriptors f */
    const int64_t *id;      /* [n] ids echoed in assignments; NULL means 0..n-1 */
} hgm_points;

/* Energy weights and temporal closeness (0.6, 0.2, 5, T = 10;
 * W^d default 1.0, R6). */
typedef struct {
    float lambda1, lambda2, lambda3, w_dummy;
    int32_t T;
} hgm_params;

/* Scene blocks: offset k covers frames [first_frame + k*stride,
 * first_frame + k*stride + window) (reading R13).  Defaults W = 60, stride 1. */
typedef struct {
    int32_t first_frame, stride, count, window;
} hgm_offsets;

/* Build the model chain: per occupied frame keep the most
 * salient point (ties: earliest input point, R-D1), nodes ordered by frame;
 * hyperedges (i, i-1, i-2) are implicit.  Also tabulates, per triple, the
 * model's frame gaps and angle constants of Eqs. 4-6 on the device.
 *   host variant: `pts` arrays are host memory; synchronous.
 *   dev  variant: `pts` arrays are device memory on `device`'s context;
 *                 runs on `stream`, returns after the handle is ready.
 * Errors: n == 0 -> EMPTY_POINT_SET; NULL arrays / F < 1 / a non-finite coordinate,
 * saliency or descriptor component / a frame outside [0, 2^26] -> INVALID_ARGUMENT
 * (saliency may be NULL: all points equally salient). */
hgm_status hgm_build_model_graph(const hgm_points *pts, int device, hgm_model **out);
hgm_status hgm_build_model_graph_dev(const hgm_points *pts, void *stream, hgm_model **out);
/* Independent chains ("Multiple points 2: creation of
 * several single point models (several second order chains), each of which is solved
 * independently"): chain `rank` keeps, per frame, the point of saliency rank `rank`
 * (0 = most salient, i.e. hgm_build_model_graph; ties: earlier input point first);
 * frames with <= rank points have no node.  Same host-memory input as
 * hgm_build_model_graph; synchronous.
 * Errors: as hgm_build_model_graph; rank < 0 -> INVALID_ARGUMENT; no frame with more
 * than `rank` points -> EMPTY_POINT_SET. */
hgm_status hgm_build_model_chain(const hgm_points *pts, int device, int32_t rank, hgm_model **out);
hgm_status hgm_model_num_nodes(const hgm_model *model, int32_t *M);
void hgm_free_model(hgm_model *model);

/* Build the scene index (§3.4): stable sort of the points by
 * frame; minnode(f) = first node with frame >= f (sentinel S, R4); and the
 * band of ordered node pairs (a, c) with 1 <= t'(c) - t'(a) <= T_max - 1
 * holding the direction of a->c and a coincidence flag.
 * T_max bounds the T of later calls.  Any T_max (and any later T) above the scene's
 * frame span is legal and means "unpruned": the band is built for
 * min(T_max, last frame + 1), which admits every pair, and calls run with
 * min(T, last frame + 1) -- the same result, no integer overflow.
 * Same host / dev split as above.
 * Errors: n == 0 -> EMPTY_POINT_SET; T_max < 1, a frame outside [0, 2^26], a non-finite
 * coordinate or descriptor component -> INVALID_ARGUMENT. */
hgm_status hgm_build_scene_index(const hgm_points *pts, int device, int32_t T_max, hgm_scene **out);
hgm_status hgm_build_scene_index_dev(const hgm_points *pts, int32_t T_max, void *stream, hgm_scene **out);
hgm_status hgm_scene_num_nodes(const hgm_scene *scene, int64_t *S);
void hgm_free_scene(hgm_scene *scene);

/* Match one model against every offset (Eqs. 10-13 at every block
 * of P:L739-743).  For offset k:
 *   E[k]        = min_z E(z)  (Eq. 1 on the chain, lambdas explicit), fp32
 *   A[k]        = sum_i U(i, z_i) of the returned z (unweighted, R14)
 *   z[k*M + i]  = caller id of the scene point matched to model node i, or -1
 *                 for the dummy; z is the lexicographically smallest optimum
 *                 of the GPU's own fp32 arithmetic (R11, R12).
 * Any of E, A, z may be NULL (not written).  Windows past the last frame are
 * legal (fewer nodes); an empty window gives the all-dummy assignment. */
hgm_status hgm_match_model_at_offsets(const hgm_model *model, const hgm_scene *scene,
                                      const hgm_params *params, const hgm_offsets *offsets,
                                      float *E, float *A, int64_t *z, void *stream);

/* Detect actions (P:L712 nearest-prototype rule, R14): for every offset k,
 *   winner[k] = smallest m attaining min_m score(m, k), or -1 if that minimum
 *               exceeds `threshold` (use +inf for none),
 *   score[k]  = that minimum, score = E (score_mode 0) or A (score_mode 1),
 *   E_all[m*count + k] = E of every pair (NULL: not written).
 * Errors: n_models == 0 -> EMPTY_POINT_SET; models of different F than the
 * scene -> DIMENSION_MISMATCH. */
hgm_status hgm_detect_actions(const hgm_model *const *models, int32_t n_models, const hgm_scene *scene,
                              const hgm_params *params, const hgm_offsets *offsets, int32_t score_mode,
                              float threshold, int32_t *winner, float *score, float *E_all, void *stream);

/* Detection with multi-chain models (f3): `chains` [n_chains] are the
 * chains of n_models models, grouped (chain_model: host [n_chains], non-decreasing,
 * every model in [0, n_models) present).  The distance of model m at offset k is the
 * mean over its chains of their score (E* for score_mode 0, A for 1, as
 * hgm_detect_actions); winner / score as hgm_detect_actions over these means (ties ->
 * lowest model); S_all (optional, [n_models][count]) receives the means.  Outputs host
 * or device.  Errors: as hgm_detect_actions; chain_model NULL / out of range / not
 * grouped -> INVALID_ARGUMENT; a model without a chain -> EMPTY_POINT_SET. */
hgm_status hgm_detect_chains(const hgm_model *const *chains, int32_t n_chains, const int32_t *chain_model,
                             int32_t n_models, const hgm_scene *scene, const hgm_params *params,
                             const hgm_offsets *offsets, int32_t score_mode, float threshold, int32_t *winner,
                             float *score, float *S_all, void *stream);

/* Streaming detection (P:L739-743 continuous processing in
 * overlapping blocks).  A stream owns a host copy of the points of the frames its
 * future windows still need; the models are borrowed (they must outlive the stream).
 * hgm_stream_create: window W, stride, score_mode and threshold as hgm_detect_actions;
 *   offsets are 0, stride, 2*stride, ... of the stream's frame clock (starting at 0).
 * hgm_stream_push: appends `pts` (host arrays; every frame in [seen, seen + n_frames),
 *   `seen` = frames pushed before; pts may be NULL or empty) and advances the clock by
 *   n_frames; then detects every offset o not yet reported whose window is complete
 *   (o + W <= seen), writing *n_out results (winner / score as hgm_detect_actions, host
 *   or device, capacity entries available) for offsets *first_offset + j * stride.
 *   Results are identical to one hgm_detect_actions call over the whole stream.
 *   Synchronous.  A push that fails (any status) leaves the stream unchanged: its frames
 *   are not consumed and the same push may be retried.
 *   Errors: NULL st / n_out / first_offset, n_frames < 0, points outside
 *   the pushed frames, capacity too small -> INVALID_ARGUMENT; F differing from the
 *   models' -> DIMENSION_MISMATCH; CUDA errors as elsewhere.  Windows without points
 *   (silent stretches) are valid and give the all-dummy result. */
typedef struct hgm_stream hgm_stream;
hgm_status hgm_stream_create(const hgm_model *const *models, int32_t n_models, const hgm_params *params,
                             int32_t window, int32_t stride, int32_t score_mode, float threshold, int32_t device,
                             hgm_stream **out);
hgm_status hgm_stream_push(hgm_stream *stream, const hgm_points *pts, int32_t n_frames, int32_t capacity,
                           int32_t *winner, float *score, int32_t *n_out, int64_t *first_offset);
void hgm_stream_free(hgm_stream *stream);

/* Recognition ("nearest prototype classifier (NPC)" with the
 * appearance distance only, P:L739-743 blocks of 60 frames; SPEC classify / split_blocks):
 * every prototype is matched against every block (block k = frames
 * [first_frame + k*stride, ... + window), the `offsets` of detect) and scored by its
 * appearance distance A (R14).
 *   block_label[k] = label[m*] of the nearest prototype m* (ties -> lowest prototype
 *                    index), -1 if its distance exceeds `threshold` (+inf: none);
 *   block_score[k] = that distance;
 *   *clip_label    = majority vote over the labelled blocks (ties -> smallest label),
 *                    -1 if no block is labelled.
 * label: host array [n_prototypes] of values in [0, n_labels), n_labels <= 4096.
 * block_label / block_score / clip_label: host or device pointers (NULL: not written).
 * Errors: as hgm_detect_actions; a label outside [0, n_labels) or n_labels out of range
 * -> INVALID_ARGUMENT. */
hgm_status hgm_classify_blocks(const hgm_model *const *prototypes, int32_t n_prototypes, const int32_t *label,
                               int32_t n_labels, const hgm_scene *scene, const hgm_params *params,
                               const hgm_offsets *blocks, float threshold, int32_t *block_label,
                               float *block_score, int32_t *clip_label, void *stream);

/* Kernel timing (CUDA events on the launch stream) for the roofline report.
 * When enabled, every call accumulates per-kernel-class device time.
 * Classes: 0 scene index (incl. K-G), 1 model graph, 2 unary table (K-U),
 * 3 recursion real states (K-DP), 4 backtrack (K-BT), 5 offset argmin (K-ARG),
 * 6 messages + dummy-form states (K-MSG), 7 reserved.  Also counts launches of
 * the library's own kernels (dp_launches = K-DP launches). */
typedef struct {
    double ms[8];
    int64_t launches[8];
    int64_t dp_candidates, dp_states, dp_launches;
} hgm_stats;
hgm_status hgm_set_profiling(int enable);
hgm_status hgm_get_stats(hgm_stats *out, int reset);

const char *hgm_last_error(void);
const char *hgm_version(void);

#ifdef __cplusplus
}
#endif
#endif /* HGM_H */
