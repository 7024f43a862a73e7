"""Thin ctypes binding of libhgm.so (include/hgm.h).  Argument marshalling only:
every step of the matching path runs in the library's CUDA kernels.  There is
no CPU fallback; if the library or a CUDA device is missing, calls raise.

Names follow the C ABI: build_model_graph, build_scene_index,
match_model_at_offsets, detect_actions.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HGM_LIB") or os.path.join(_HERE, "lib", "libhgm.so")  # HGM_LIB: A/B builds

STATUS = {0: "HGM_OK", 1: "HGM_ERR_EMPTY_POINT_SET", 2: "HGM_ERR_DIMENSION_MISMATCH",
          3: "HGM_ERR_INVALID_ARGUMENT", 4: "HGM_ERR_OUT_OF_MEMORY", 5: "HGM_ERR_CUDA"}

EXPORTS = ("hgm_stream_create", "hgm_stream_push", "hgm_stream_free", "hgm_build_model_graph", "hgm_build_model_graph_dev", "hgm_build_model_chain", "hgm_detect_chains", "hgm_model_num_nodes", "hgm_free_model",
           "hgm_build_scene_index", "hgm_build_scene_index_dev", "hgm_scene_num_nodes", "hgm_free_scene",
           "hgm_match_model_at_offsets", "hgm_detect_actions", "hgm_classify_blocks", "hgm_set_profiling", "hgm_get_stats",
           "hgm_last_error", "hgm_version")


class HGMError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class _Points(C.Structure):
    _fields_ = [("n", C.c_int64), ("F", C.c_int32), ("frame", C.c_void_p), ("x", C.c_void_p), ("y", C.c_void_p),
                ("saliency", C.c_void_p), ("feat", C.c_void_p), ("id", C.c_void_p)]


class Params(C.Structure):
    """Energy weights and temporal closeness T."""
    _fields_ = [("lambda1", C.c_float), ("lambda2", C.c_float), ("lambda3", C.c_float), ("w_dummy", C.c_float),
                ("T", C.c_int32)]

    @classmethod
    def make(cls, lambda1=0.6, lambda2=0.2, lambda3=5.0, w_dummy=1.0, T=10):
        return cls(lambda1, lambda2, lambda3, w_dummy, int(T))


class Offsets(C.Structure):
    _fields_ = [("first_frame", C.c_int32), ("stride", C.c_int32), ("count", C.c_int32), ("window", C.c_int32)]


class Stats(C.Structure):
    _fields_ = [("ms", C.c_double * 8), ("launches", C.c_int64 * 8), ("dp_candidates", C.c_int64),
                ("dp_states", C.c_int64), ("dp_launches", C.c_int64)]


_lib = None


def lib():
    """Load libhgm.so; raise loudly if it is missing (no fallback path exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"libhgm.so not built at {LIB_PATH}; run __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        vp, P = C.c_void_p, C.POINTER
        L.hgm_build_model_graph.argtypes = [P(_Points), C.c_int, P(vp)]
        L.hgm_stream_create.argtypes = [P(vp), C.c_int32, P(Params), C.c_int32, C.c_int32, C.c_int32, C.c_float,
                                        C.c_int32, P(vp)]
        L.hgm_stream_push.argtypes = [vp, P(_Points), C.c_int32, C.c_int32, vp, vp, P(C.c_int32), P(C.c_int64)]
        L.hgm_stream_free.argtypes = [vp]
        L.hgm_stream_free.restype = None
        L.hgm_build_model_chain.argtypes = [P(_Points), C.c_int, C.c_int32, P(vp)]
        L.hgm_detect_chains.argtypes = [P(vp), C.c_int32, vp, C.c_int32, vp, P(Params), P(Offsets), C.c_int32,
                                        C.c_float, vp, vp, vp, vp]
        L.hgm_build_model_graph_dev.argtypes = [P(_Points), vp, P(vp)]
        L.hgm_model_num_nodes.argtypes = [vp, P(C.c_int32)]
        L.hgm_free_model.argtypes = [vp]
        L.hgm_free_model.restype = None
        L.hgm_build_scene_index.argtypes = [P(_Points), C.c_int, C.c_int32, P(vp)]
        L.hgm_build_scene_index_dev.argtypes = [P(_Points), C.c_int32, vp, P(vp)]
        L.hgm_scene_num_nodes.argtypes = [vp, P(C.c_int64)]
        L.hgm_free_scene.argtypes = [vp]
        L.hgm_free_scene.restype = None
        L.hgm_match_model_at_offsets.argtypes = [vp, vp, P(Params), P(Offsets), vp, vp, vp, vp]
        L.hgm_detect_actions.argtypes = [P(vp), C.c_int32, vp, P(Params), P(Offsets), C.c_int32, C.c_float, vp, vp,
                                         vp, vp]
        L.hgm_classify_blocks.argtypes = [P(vp), C.c_int32, vp, C.c_int32, vp, P(Params), P(Offsets), C.c_float,
                                          vp, vp, vp, vp]
        L.hgm_set_profiling.argtypes = [C.c_int]
        L.hgm_get_stats.argtypes = [P(Stats), C.c_int]
        L.hgm_last_error.restype = C.c_char_p
        L.hgm_version.restype = C.c_char_p
        _lib = L
    return _lib


def _check(st):
    if st != 0:
        raise HGMError(st, lib().hgm_last_error().decode())


def _is_torch(a):
    return type(a).__module__.startswith("torch")


def _ptr(a):
    if a is None:
        return None
    if _is_torch(a):
        return a.data_ptr()
    return a.ctypes.data


class _HostPoints:
    """Contiguous typed host copies of a point set (numpy), kept alive with the struct."""

    def __init__(self, pts):
        self.frame = np.ascontiguousarray(pts.frame, dtype=np.int32)
        self.x = np.ascontiguousarray(pts.x, dtype=np.float32)
        self.y = np.ascontiguousarray(pts.y, dtype=np.float32)
        sal = getattr(pts, "saliency", None)
        self.sal = None if sal is None else np.ascontiguousarray(sal, dtype=np.float32)
        self.feat = np.ascontiguousarray(pts.feat, dtype=np.float32)
        pid = getattr(pts, "id", None)
        self.id = None if pid is None else np.ascontiguousarray(pid, dtype=np.int64)
        n = int(self.frame.shape[0])
        F = int(self.feat.shape[1]) if self.feat.ndim == 2 else 0
        self.s = _Points(n, F, _ptr(self.frame), _ptr(self.x), _ptr(self.y), _ptr(self.sal), _ptr(self.feat),
                         _ptr(self.id))


class DevicePoints:
    """A point set resident in HBM (torch CUDA tensors): frame int32, x/y/saliency
    float32, feat float32 [n, F] row-major, id int64 or None."""

    def __init__(self, frame, x, y, saliency, feat, id=None):
        self.frame, self.x, self.y, self.saliency, self.feat, self.id = frame, x, y, saliency, feat, id

    @classmethod
    def from_host(cls, pts, device="cuda", non_blocking=False, pinned=False):
        import torch

        def up(a, dt):
            t = torch.from_numpy(np.ascontiguousarray(a).astype(dt, copy=False))
            if pinned:
                t = t.pin_memory()
            return t.to(device, non_blocking=non_blocking)

        pid = getattr(pts, "id", None)
        return cls(up(pts.frame, np.int32), up(pts.x, np.float32), up(pts.y, np.float32),
                   up(pts.saliency, np.float32), up(pts.feat, np.float32), None if pid is None else up(pid, np.int64))

    def cstruct(self):
        n = int(self.frame.shape[0])
        F = int(self.feat.shape[1])
        return _Points(n, F, _ptr(self.frame), _ptr(self.x), _ptr(self.y), _ptr(self.saliency), _ptr(self.feat),
                       _ptr(self.id))


def _stream_ptr(stream):
    if stream is None:
        try:
            import torch

            return torch.cuda.current_stream().cuda_stream
        except Exception:
            return None
    return stream if isinstance(stream, int) else stream.cuda_stream


class Model:
    """Handle of a model chain in HBM (hgm_build_model_graph)."""

    def __init__(self, handle):
        self.h = C.c_void_p(handle)

    @property
    def M(self):
        m = C.c_int32()
        _check(lib().hgm_model_num_nodes(self.h, C.byref(m)))
        return m.value

    def __del__(self):
        if getattr(self, "h", None) and self.h.value and _lib is not None:
            _lib.hgm_free_model(self.h)
            self.h = None


class Scene:
    """Handle of a scene index in HBM (hgm_build_scene_index)."""

    def __init__(self, handle, T_max):
        self.h = C.c_void_p(handle)
        self.T_max = T_max

    @property
    def S(self):
        s = C.c_int64()
        _check(lib().hgm_scene_num_nodes(self.h, C.byref(s)))
        return s.value

    def __del__(self):
        if getattr(self, "h", None) and self.h.value and _lib is not None:
            _lib.hgm_free_scene(self.h)
            self.h = None


def build_model_graph(points, device: int = 0, stream=None) -> Model:
    """Model chain: host point sets are copied; DevicePoints stay on the GPU."""
    out = C.c_void_p()
    if isinstance(points, DevicePoints):
        _check(lib().hgm_build_model_graph_dev(C.byref(points.cstruct()), _stream_ptr(stream), C.byref(out)))
    else:
        hp = _HostPoints(points)
        _check(lib().hgm_build_model_graph(C.byref(hp.s), int(device), C.byref(out)))
    return Model(out.value)


def build_model_chains(points, n_chains: int, device: int = 0) -> list:
    """Chains 0..n_chains-1 of the independent-chains model:
    chain r keeps each frame's point of saliency rank r.  Ranks no frame reaches
    are skipped (the list may be shorter than n_chains)."""
    hp = _HostPoints(points)
    out = []
    for r in range(int(n_chains)):
        h = C.c_void_p()
        st = lib().hgm_build_model_chain(C.byref(hp.s), int(device), int(r), C.byref(h))
        if st == 1:  # HGM_ERR_EMPTY_POINT_SET: no frame has more than r points
            break
        _check(st)
        out.append(Model(h.value))
    return out


def build_scene_index(points, device: int = 0, T_max: int = 10, stream=None) -> Scene:
    """Scene index."""
    out = C.c_void_p()
    if isinstance(points, DevicePoints):
        _check(lib().hgm_build_scene_index_dev(C.byref(points.cstruct()), int(T_max), _stream_ptr(stream),
                                               C.byref(out)))
    else:
        hp = _HostPoints(points)
        _check(lib().hgm_build_scene_index(C.byref(hp.s), int(device), int(T_max), C.byref(out)))
    return Scene(out.value, T_max)


def _params(params):
    if isinstance(params, Params):
        return params
    return Params.make(**(params or {}))


@dataclass
class MatchResult:
    E: object  # [count] float32
    A: object  # [count] float32
    z: object  # [count, M] int64 caller ids, -1 = dummy


def match_model_at_offsets(model: Model, scene: Scene, params=None, first_frame=0, stride=1, count=1, window=60,
                           device_out: bool = True, stream=None) -> MatchResult:
    """E*, A and the assignment of one model at every offset (Eqs. 10-13)."""
    M = model.M
    if device_out:
        import torch

        E = torch.empty(count, dtype=torch.float32, device="cuda")
        A = torch.empty(count, dtype=torch.float32, device="cuda")
        z = torch.empty((count, M), dtype=torch.int64, device="cuda")
    else:
        E = np.empty(count, np.float32)
        A = np.empty(count, np.float32)
        z = np.empty((count, M), np.int64)
    o = Offsets(int(first_frame), int(stride), int(count), int(window))
    _check(lib().hgm_match_model_at_offsets(model.h, scene.h, C.byref(_params(params)), C.byref(o), _ptr(E), _ptr(A),
                                            _ptr(z), _stream_ptr(stream)))
    return MatchResult(E, A, z)


@dataclass
class DetectResult:
    winner: object  # [count] int32, -1 above threshold
    score: object  # [count] float32
    E_all: object  # [n_models, count] float32 or None


def detect_actions(models, scene: Scene, params=None, first_frame=0, stride=1, count=1, window=60, score_mode=0,
                   threshold=math.inf, want_E_all=False, device_out=True, out=None, stream=None) -> DetectResult:
    """Per-offset nearest-model detection.  `out` may supply
    preallocated (winner, score, E_all) buffers."""
    nm = len(models)
    if out is not None:
        winner, score, E_all = out
    elif device_out:
        import torch

        winner = torch.empty(count, dtype=torch.int32, device="cuda")
        score = torch.empty(count, dtype=torch.float32, device="cuda")
        E_all = torch.empty((nm, count), dtype=torch.float32, device="cuda") if want_E_all else None
    else:
        winner = np.empty(count, np.int32)
        score = np.empty(count, np.float32)
        E_all = np.empty((nm, count), np.float32) if want_E_all else None
    handles = (C.c_void_p * nm)(*[m.h.value for m in models])
    o = Offsets(int(first_frame), int(stride), int(count), int(window))
    _check(lib().hgm_detect_actions(handles, nm, scene.h, C.byref(_params(params)), C.byref(o), int(score_mode),
                                    float(threshold), _ptr(winner), _ptr(score), _ptr(E_all), _stream_ptr(stream)))
    return DetectResult(winner, score, E_all)


def detect_chains(chains, chain_model, n_models, scene: Scene, params=None, first_frame=0, stride=1, count=1,
                  window=60, score_mode=0, threshold=math.inf, want_S_all=False, device_out=True,
                  stream=None) -> DetectResult:
    """Detection with multi-chain models (hgm_detect_chains): a
    model's distance is the mean of its chains' scores.  `E_all` of the result holds
    the per-model means when want_S_all."""
    nc = len(chains)
    cm = np.ascontiguousarray(chain_model, dtype=np.int32)
    if cm.shape != (nc,):
        raise ValueError("chain_model must have one entry per chain")
    if device_out:
        import torch

        winner = torch.empty(count, dtype=torch.int32, device="cuda")
        score = torch.empty(count, dtype=torch.float32, device="cuda")
        S_all = torch.empty((n_models, count), dtype=torch.float32, device="cuda") if want_S_all else None
    else:
        winner = np.empty(count, np.int32)
        score = np.empty(count, np.float32)
        S_all = np.empty((n_models, count), np.float32) if want_S_all else None
    handles = (C.c_void_p * nc)(*[m.h.value for m in chains])
    o = Offsets(int(first_frame), int(stride), int(count), int(window))
    _check(lib().hgm_detect_chains(handles, nc, cm.ctypes.data, int(n_models), scene.h, C.byref(_params(params)),
                                   C.byref(o), int(score_mode), float(threshold), _ptr(winner), _ptr(score),
                                   _ptr(S_all), _stream_ptr(stream)))
    return DetectResult(winner, score, S_all)


class Stream:
    """Streaming detection (hgm_stream_*): push frames in order,
    get the offsets whose windows completed.  The models must outlive the stream."""

    def __init__(self, models, params=None, window=60, stride=1, score_mode=0, threshold=math.inf, device=0):
        self.models = list(models)  # keep the handles alive
        h = C.c_void_p()
        handles = (C.c_void_p * len(self.models))(*[m.h.value for m in self.models])
        _check(lib().hgm_stream_create(handles, len(self.models), C.byref(_params(params)), int(window), int(stride),
                                       int(score_mode), float(threshold), int(device), C.byref(h)))
        self.h = h
        self.window, self.stride = int(window), int(stride)
        self.seen, self.o_next = 0, 0  # mirrors of the library's stream state (output sizing)

    def push(self, points, n_frames: int):
        """Append `points` (frames in [seen, seen + n_frames), or None) and return
        (first_offset, winner int32[n], score float32[n]) for the completed offsets.
        A failed push leaves the stream unchanged."""
        seen1 = self.seen + int(n_frames)
        cap = max(0, (seen1 - self.window - self.o_next) // self.stride + 1) + 1  # the whole backlog
        winner = np.empty(cap, np.int32)
        score = np.empty(cap, np.float32)
        n = C.c_int32()
        first = C.c_int64()
        hp = _HostPoints(points) if points is not None and points.n > 0 else None
        _check(lib().hgm_stream_push(self.h, C.byref(hp.s) if hp else None, int(n_frames), cap, winner.ctypes.data,
                                     score.ctypes.data, C.byref(n), C.byref(first)))
        self.seen = seen1
        self.o_next = int(first.value) + n.value * self.stride
        return int(first.value), winner[: n.value].copy(), score[: n.value].copy()

    def __del__(self):
        if getattr(self, "h", None) and self.h.value and _lib is not None:
            _lib.hgm_stream_free(self.h)
            self.h = None


@dataclass
class ClassifyResult:
    block_label: object  # int32 [count]
    block_score: object  # float32 [count]: appearance distance of the nearest prototype
    clip_label: int  # majority vote, -1 if no block is labelled


def classify_blocks(prototypes, labels, scene: Scene, params=None, first_frame=0, stride=60, count=1, window=60,
                    threshold=math.inf, n_labels=None, stream=None) -> ClassifyResult:
    """Nearest-prototype recognition per scene block + majority vote
    (hgm_classify_blocks).  Host outputs."""
    nm = len(prototypes)
    lab = np.ascontiguousarray(labels, dtype=np.int32)
    if lab.shape != (nm,):
        raise ValueError("labels must have one entry per prototype")
    n_labels = int(lab.max()) + 1 if n_labels is None else int(n_labels)
    bl = np.empty(count, np.int32)
    bs = np.empty(count, np.float32)
    cl = np.empty(1, np.int32)
    handles = (C.c_void_p * nm)(*[m.h.value for m in prototypes])
    o = Offsets(int(first_frame), int(stride), int(count), int(window))
    _check(lib().hgm_classify_blocks(handles, nm, lab.ctypes.data, n_labels, scene.h, C.byref(_params(params)),
                                     C.byref(o), float(threshold), _ptr(bl), _ptr(bs), _ptr(cl),
                                     _stream_ptr(stream)))
    return ClassifyResult(bl, bs, int(cl[0]))


def set_profiling(enable: bool = True):
    _check(lib().hgm_set_profiling(int(bool(enable))))


def get_stats(reset: bool = False) -> dict:
    s = Stats()
    _check(lib().hgm_get_stats(C.byref(s), int(bool(reset))))
    names = ("scene", "model", "unary", "dp", "backtrack", "argmin", "unused", "reserved")
    return dict(ms={n: s.ms[i] for i, n in enumerate(names)},
                launches={n: s.launches[i] for i, n in enumerate(names)}, dp_launches=s.dp_launches)


def version() -> str:
    return lib().hgm_version().decode()
