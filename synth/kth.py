"""KTH-shaped synthetic point sets (SURVEY.md §8(d) "Synthetic KTH-shaped inputs").

Everything here is drawing random numbers; nothing computes the matching energy,
selects model nodes or sorts the scene (those are the method, implemented
separately by `oracle/` and by the CUDA library).

Randomness: numpy PCG64 streams keyed by SeedSequence([crc32(config), *stream]),
so every (config, clip, segment, stream) draws independently of the others and
a rank can regenerate any scene segment on its own (multi-GPU bench).
"""
from __future__ import annotations

import zlib
from dataclasses import dataclass, field

import numpy as np

FRAME_W = 160  # PAPER.md L707 (§4): KTH images are 160x120
FRAME_H = 120
F_KTH = 162  # PAPER.md L345 (§3.3): 162 components for HoG/HoF
N_CLASSES = 6  # PAPER.md L705 (§4): six KTH actions
CODEBOOK = 16  # prototypes per class codebook


@dataclass
class Points:
    """A raw interest-point set: one row per detected point (S:L20-24 shape)."""

    frame: np.ndarray  # int32 [n] >= 0
    x: np.ndarray  # float32 [n], integer-valued pixels
    y: np.ndarray  # float32 [n]
    saliency: np.ndarray  # float32 [n]
    feat: np.ndarray  # float32 [n, F]
    id: np.ndarray | None = None  # int64 [n] ids echoed in assignments

    @property
    def n(self) -> int:
        return int(self.frame.shape[0])

    @property
    def F(self) -> int:
        return int(self.feat.shape[1])

    def take(self, idx) -> "Points":
        idx = np.asarray(idx)
        return Points(
            self.frame[idx].copy(),
            self.x[idx].copy(),
            self.y[idx].copy(),
            self.saliency[idx].copy(),
            self.feat[idx].copy(),
            None if self.id is None else self.id[idx].copy(),
        )

    def ids(self) -> np.ndarray:
        return np.arange(self.n, dtype=np.int64) if self.id is None else self.id


def _rng(config: str, *stream: int) -> np.random.Generator:
    key = zlib.crc32(config.encode())
    return np.random.default_rng(np.random.SeedSequence([key, *[int(s) for s in stream]]))


def _unit_nonneg(rng: np.random.Generator, n: int, F: int) -> np.ndarray:
    v = np.abs(rng.standard_normal((n, F)))
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    return v.astype(np.float32)


def _renorm_nonneg(v: np.ndarray) -> np.ndarray:
    v = np.maximum(v, 0.0)
    nrm = np.linalg.norm(v, axis=1, keepdims=True)
    nrm[nrm == 0] = 1.0
    return (v / nrm).astype(np.float32)


def _clip_px(x, y):
    return (
        np.clip(np.rint(x), 0, FRAME_W - 1).astype(np.float32),
        np.clip(np.rint(y), 0, FRAME_H - 1).astype(np.float32),
    )


def codebook(cls: int, F: int, config: str = "codebook") -> np.ndarray:
    """Per-class prototype descriptors (non-negative, unit L2)."""
    return _unit_nonneg(_rng(config, 7, cls, F), CODEBOOK, F)


def gen_model(cls: int, n_frames: int, pts_per_frame: int, F: int, config: str, stream: int,
              gap2_prob: float = 0.15, feat_sigma: float = 0.1) -> Points:
    """A model action clip: an actor trajectory with `pts_per_frame` raw points
    in each of `n_frames` occupied frames (centre random walk N(0,2^2) px/frame,
    body-part offsets N(0,15^2) px, integer pixels).  Occupied frames are spaced
    by gaps of 1 or 2 frames (empty model frames)."""
    rng = _rng(config, 1, cls, stream)
    gaps = np.where(rng.random(n_frames - 1) < gap2_prob, 2, 1) if n_frames > 1 else np.zeros(0, int)
    frames = np.concatenate([[0], np.cumsum(gaps)]).astype(np.int32)
    n_steps = int(frames[-1]) + 1
    centre = np.cumsum(rng.normal(0.0, 2.0, size=(n_steps, 2)), axis=0)
    centre += np.array([rng.uniform(50, 110), rng.uniform(35, 85)])
    fr = np.repeat(frames, pts_per_frame)
    c = centre[fr]
    off = rng.normal(0.0, 15.0, size=(fr.shape[0], 2))
    x, y = _clip_px(c[:, 0] + off[:, 0], c[:, 1] + off[:, 1])
    cb = codebook(cls, F)
    k = rng.integers(0, CODEBOOK, size=fr.shape[0])
    feat = _renorm_nonneg(cb[k] + rng.normal(0.0, feat_sigma, size=(fr.shape[0], F)))
    sal = rng.random(fr.shape[0]).astype(np.float32)
    return Points(fr.astype(np.int32), x, y, sal, feat)


def gen_clutter(n_frames: int, f0: int, rho: float, F: int, rng: np.random.Generator,
                exact_count: int | None = None) -> Points:
    """Poisson(rho) clutter points per frame in [f0, f0+n_frames), uniform integer
    pixels, random non-negative unit descriptors."""
    if exact_count is None:
        counts = rng.poisson(rho, size=n_frames)
        fr = np.repeat(np.arange(f0, f0 + n_frames), counts)
    else:
        fr = np.sort(rng.integers(f0, f0 + n_frames, size=exact_count))
    n = fr.shape[0]
    x = rng.integers(0, FRAME_W, size=n).astype(np.float32)
    y = rng.integers(0, FRAME_H, size=n).astype(np.float32)
    return Points(fr.astype(np.int32), x, y, rng.random(n).astype(np.float32), _unit_nonneg(rng, n, F))


def gen_planted(model: Points, start: int, T: int, rng: np.random.Generator,
                feat_sigma: float = 0.02, jitter: int = 1, warp: bool = True) -> Points:
    """A warped copy of ALL raw model points: occupied-frame gaps g+d,
    d in {-1,0,0,+1}, gaps >= 1, two consecutive gaps summing to <= T-1;
    integer translation, +-jitter px, descriptor noise N(0, feat_sigma^2)
    renormalised."""
    uf = np.unique(model.frame)
    gaps = np.diff(uf).astype(np.int64)
    if warp and gaps.size:
        d = rng.choice(np.array([-1, 0, 0, 1]), size=gaps.size)
        gaps = np.maximum(gaps + d, 1)
    for k in range(1, gaps.size):  # keep the planted chain temporally close
        while gaps[k] + gaps[k - 1] > max(T - 1, 2) and gaps[k] > 1:
            gaps[k] -= 1
    new_uf = start + np.concatenate([[0], np.cumsum(gaps)]).astype(np.int64)
    remap = dict(zip(uf.tolist(), new_uf.tolist()))
    fr = np.array([remap[int(f)] for f in model.frame], dtype=np.int32)
    cx = model.x.mean()
    cy = model.y.mean()
    dx = rng.integers(int(-cx) + 20, int(FRAME_W - cx) - 20 + 1) if FRAME_W - 40 > 0 else 0
    dy = rng.integers(int(-cy) + 15, int(FRAME_H - cy) - 15 + 1) if FRAME_H - 30 > 0 else 0
    jx = rng.integers(-jitter, jitter + 1, size=model.n) if jitter else 0
    jy = rng.integers(-jitter, jitter + 1, size=model.n) if jitter else 0
    x, y = _clip_px(model.x + dx + jx, model.y + dy + jy)
    feat = model.feat + (rng.normal(0.0, feat_sigma, size=model.feat.shape) if feat_sigma > 0 else 0.0)
    feat = _renorm_nonneg(feat) if feat_sigma > 0 else model.feat.copy()
    sal = rng.random(model.n).astype(np.float32)
    return Points(fr, x, y, sal, feat)


def concat_points(parts: list[Points]) -> Points:
    parts = [p for p in parts if p.n > 0] or parts[:1]
    return Points(
        np.concatenate([p.frame for p in parts]).astype(np.int32),
        np.concatenate([p.x for p in parts]).astype(np.float32),
        np.concatenate([p.y for p in parts]).astype(np.float32),
        np.concatenate([p.saliency for p in parts]).astype(np.float32),
        np.concatenate([p.feat for p in parts]).astype(np.float32),
    )


def _span(model: Points) -> int:
    return int(model.frame.max() - model.frame.min()) + 1


@dataclass
class Workload:
    """One benchmark / parity configuration."""

    name: str
    models: list[Points]
    scenes: list[Points]  # C2 has 25 clips; others one scene
    window: int
    stride: int
    first_frame: int
    count: list[int]  # offsets per scene
    lambda1: float = 0.6  # PAPER.md L710 (§4)
    lambda2: float = 0.2
    lambda3: float = 5.0
    w_dummy: float = 1.0  # SURVEY §8c A6 / S:L192
    T: int = 10
    first: list[int] = field(default_factory=list)  # first offset per scene

    def params(self) -> dict:
        return dict(lambda1=self.lambda1, lambda2=self.lambda2, lambda3=self.lambda3,
                    w_dummy=self.w_dummy, T=self.T)

    @property
    def n_pairs(self) -> int:
        return len(self.models) * sum(self.count)


def _scene_from_segments(config: str, n_frames: int, seg_len: int, rho: float, F: int, T: int,
                         models: list[Points], frame_range: tuple[int, int] | None,
                         plants_per_seg: int = 1, cls_of_seg=None) -> Points:
    """Scene of n_frames built from independent seg_len-frame segments, each
    seeded by its index (so any frame range can be regenerated alone)."""
    lo, hi = (0, n_frames) if frame_range is None else frame_range
    parts = []
    for s in range(max(0, lo // seg_len), min((n_frames + seg_len - 1) // seg_len, (hi + seg_len - 1) // seg_len)):
        rng = _rng(config, 2, s)
        f0 = s * seg_len
        nf = min(seg_len, n_frames - f0)
        parts.append(gen_clutter(nf, f0, rho, F, rng))
        # planted instances inside the segment (non-overlapping slots)
        slot = nf // max(plants_per_seg, 1)
        for k in range(plants_per_seg):
            cls = (cls_of_seg(s) if cls_of_seg is not None else int(rng.integers(0, len(models))))
            m = models[cls % len(models)]
            room = slot - (_span(m) + _span(m) // 2 + 2)
            if room <= 0:
                continue
            start = f0 + k * slot + int(rng.integers(0, room))
            parts.append(gen_planted(m, start, T, rng))
    sc = concat_points(parts)
    keep = np.nonzero((sc.frame >= lo) & (sc.frame < hi))[0]
    return sc.take(keep)


CONFIGS = ("C0", "C1", "C2", "C3", "C4")


def make_workload(name: str, seed: int = 0, T: int | None = None, frame_range=None,
                  n_frames: int | None = None, rho: float | None = None) -> Workload:
    """Build one of the SURVEY.md §8(d) configurations.

    C0 tiny  : 1 model M=8 (1 pt/frame, F=8), scene 40 pts over 20 frames, T=5, one window.
    C1       : 1 model (60 raw pts, 2/frame, 30 frames) vs a 600-frame clip, rho=2.5,
               4 planted copies, W=60 stride 1 (541 offsets).
    C2       : 6 models x 25 clips of 600 frames, rho=5, 2 planted per clip, W=60 stride 1.
    C3       : one long scene (25,000 frames, rho=4, one planted instance per 200 frames),
               6 models, W=60 stride 1.  `frame_range` regenerates a slice (sharding).
    C4       : 6 models of 200 frames (1 pt/frame) vs 4,000 frames at rho=4, W=400, stride 10.
    """
    cfg = f"{name}:{seed}"
    if name == "C0":
        T = 5 if T is None else T
        F = 8
        model = gen_model(0, 8, 1, F, cfg, 0, gap2_prob=0.0)
        rng = _rng(cfg, 3)
        clutter = gen_clutter(20, 0, 0.0, F, rng, exact_count=32)
        # a warped copy of an 8-frame chain spans at most 15 frames: start in [0, 5]
        planted = gen_planted(model, int(rng.integers(0, 6)), T, rng, feat_sigma=0.05)
        scene = concat_points([clutter, planted])
        return Workload(name, [model], [scene], window=20, stride=1, first_frame=0, count=[1],
                        T=T, first=[0])
    if name == "C1":
        T = 10 if T is None else T
        model = gen_model(0, 30, 2, F_KTH, cfg, 0)
        nf = 600 if n_frames is None else n_frames
        scene = _scene_from_segments(cfg, nf, 150, 2.5 if rho is None else rho, F_KTH, T,
                                     [model], frame_range)
        return Workload(name, [model], [scene], 60, 1, 0, [nf - 60 + 1], T=T, first=[0])
    if name == "C2":
        T = 10 if T is None else T
        models = [gen_model(c, 30, 2, F_KTH, cfg, 0) for c in range(N_CLASSES)]
        scenes = []
        for clip in range(25):
            scenes.append(_scene_from_segments(f"{cfg}:clip{clip}", 600, 300,
                                               5.0 if rho is None else rho, F_KTH, T, models, None,
                                               cls_of_seg=lambda s, c=clip: c % N_CLASSES))
        return Workload(name, models, scenes, 60, 1, 0, [541] * 25, T=T, first=[0] * 25)
    if name == "C3":
        T = 10 if T is None else T
        models = [gen_model(c, 30, 2, F_KTH, cfg, 0) for c in range(N_CLASSES)]
        nf = 25000 if n_frames is None else n_frames
        scene = _scene_from_segments(cfg, nf, 200, 4.0 if rho is None else rho, F_KTH, T, models,
                                     frame_range)
        return Workload(name, models, [scene], 60, 1, 0, [nf - 60 + 1], T=T, first=[0])
    if name == "C4":
        T = 20 if T is None else T
        models = [gen_model(c, 200, 1, F_KTH, cfg, 0, gap2_prob=0.0) for c in range(N_CLASSES)]
        nf = 4000 if n_frames is None else n_frames
        scene = _scene_from_segments(cfg, nf, 500, 4.0 if rho is None else rho, F_KTH, T, models,
                                     frame_range)
        return Workload(name, models, [scene], 400, 10, 0, [(nf - 400) // 10 + 1], T=T, first=[0])
    raise ValueError(f"unknown config {name}")


@dataclass
class RecognitionSet:
    """A prototype dictionary and one scene clip cut into blocks."""

    prototypes: list[Points]
    labels: np.ndarray  # int32 [n_prototypes]
    scene: Points
    block: int  # block length in frames (= window)
    stride: int
    count: int  # number of blocks
    truth: np.ndarray  # int32 [count]: class planted in block k
    T: int = 10

    def params(self) -> dict:
        return dict(lambda1=0.6, lambda2=0.2, lambda3=5.0, w_dummy=1.0, T=self.T)


def make_recognition(seed: int = 0, n_classes: int = N_CLASSES, protos_per_class: int = 2, count: int = 8,
                     block: int = 60, model_frames: int = 30, pts_per_frame: int = 2, F: int = F_KTH,
                     rho: float = 5.0, T: int = 10, exact: bool = False, clip_class: int | None = None,
                     class_of_block=None) -> RecognitionSet:
    """Prototypes: `protos_per_class` sub-sequence models per class (PAPER.md L712:
    'augmented the number of model graph prototypes'), labels = class.  Scene:
    `count` consecutive blocks of `block` frames (L739: 60-frame blocks), Poisson
    clutter plus one planted instance of prototype (class c, stream 0) per block,
    c = clip_class, or class_of_block(k), or drawn.  exact=True plants unwarped,
    noise-free, jitter-free copies (distance 0 to their prototype)."""
    cfg = f"R:{seed}"
    protos, labels = [], []
    for c in range(n_classes):
        for s in range(protos_per_class):
            protos.append(gen_model(c, model_frames, pts_per_frame, F, cfg, s,
                                    gap2_prob=0.0 if exact else 0.15))
            labels.append(c)
    rng = _rng(cfg, 9)
    parts, truth = [], []
    for k in range(count):
        c = clip_class if clip_class is not None else (
            class_of_block(k) if class_of_block is not None else int(rng.integers(0, n_classes)))
        truth.append(c)
        f0 = k * block
        parts.append(gen_clutter(block, f0, rho, F, rng))
        m = protos[c * protos_per_class]
        room = block - (_span(m) + _span(m) // 2 + 2) if not exact else block - _span(m)
        start = f0 + int(rng.integers(0, max(room, 0) + 1))
        if exact:
            parts.append(Points((m.frame - m.frame.min() + start).astype(np.int32), m.x.copy(), m.y.copy(),
                                m.saliency.copy(), m.feat.copy()))
        else:
            parts.append(gen_planted(m, start, T, rng))
    return RecognitionSet(protos, np.array(labels, np.int32), concat_points(parts), block, block, count,
                          np.array(truth, np.int32), T)


def make_single(seed: int = 0, n_frames: int = 723, n_nodes: int = 754, model_frames: int = 30, F: int = F_KTH,
                T: int = 10, plant: bool = True) -> Workload:
    """The paper's single-instance regime (Table 3): ONE model of
    30 nodes (1 point per frame) against a whole scene video of `n_nodes` nodes over
    `n_frames` frames (754 / 723), one window covering the whole video.  Scene: one
    clutter point in every frame, the remaining n_nodes - n_frames points in random
    frames, and one planted warped copy of the model; the planted points replace
    clutter so the node count stays n_nodes (up to the model's size)."""
    cfg = f"S:{seed}"
    model = gen_model(0, model_frames, 1, F, cfg, 0)
    rng = _rng(cfg, 4)
    span = _span(model)
    start = int(rng.integers(0, max(n_frames - 2 * span, 0) + 1))
    planted = gen_planted(model, start, T, rng) if plant else gen_clutter(0, 0, 0.0, F, rng, exact_count=0)
    n_extra = max(n_nodes - n_frames - planted.n, 0)
    fr = np.sort(np.concatenate([np.arange(n_frames), rng.integers(0, n_frames, size=n_extra)]))
    clutter = gen_clutter(n_frames, 0, 0.0, F, rng, exact_count=fr.shape[0])
    clutter.frame[:] = fr
    scene = concat_points([clutter, planted])
    return Workload("single", [model], [scene], window=n_frames, stride=1, first_frame=0, count=[1], T=T,
                    first=[0])
