"""CPU ORACLE for the hypergraph-matching hot path.  TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py` (its `cpu_baseline` leg
and `--impl reference`) may import this package.  The product
(`paper_1505_00581_b200`, `libhgm.so`) never imports, links or calls it, and
this package imports nothing from the product.  The only code both sides share
is the seeded generator in `synth/`, which holds none of the method's arithmetic.

Contents (each cites the passage it transcribes):
  * `model_chain`   -- one most-salient point per model frame (§2.1)
  * `scene_sorted`  -- frame-sorted scene, stable (§3.4)
  * `window_range`  -- nodes of the block [o, o+W) (reading A13)
  * `match`, `match_batch`, `detect` -- the exact DP of Eqs. 10-13 in fp64 (C, hgm_oracle.c)
  * `energy`, `feasible`, `brute` -- Eq. 1 and a DFS enumerator (C, hgm_brute.c)
  * `exhaustive` (module) -- pure-Python (S+1)^M enumeration for the tiniest cases

Parity: pinned by tests/test_oracle_*.py; see DESIGN.md §4.  Nothing here is
"parity unpinned".
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_SRC = [os.path.join(_HERE, "hgm_oracle.c"), os.path.join(_HERE, "hgm_brute.c")]
_lib = None


def build(force: bool = False) -> str:
    """Compile the C oracle (plain gcc, -O2, no fast-math so fp64 is IEEE)."""
    newest = max(os.path.getmtime(s) for s in _SRC)
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < newest:
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-fPIC", "-shared", "-fno-fast-math",
                               "-ffp-contract=off", *_SRC, "-o", tmp, "-lm", "-lpthread"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


class _Params(C.Structure):
    _fields_ = [("lambda1", C.c_double), ("lambda2", C.c_double), ("lambda3", C.c_double),
                ("w_dummy", C.c_double), ("T", C.c_int)]


class _Set(C.Structure):  # or_model / or_scene share one layout
    _fields_ = [("n", C.c_int), ("F", C.c_int), ("t", C.POINTER(C.c_int)),
                ("x", C.POINTER(C.c_double)), ("y", C.POINTER(C.c_double)),
                ("f", C.POINTER(C.c_double))]


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB_PATH)
        P, S = C.POINTER(_Params), C.POINTER(_Set)
        dp, ip = C.POINTER(C.c_double), C.POINTER(C.c_int)
        L.or_match.argtypes = [S, S, P, dp, dp, dp, ip]
        L.or_match_batch.argtypes = [S, S, P, C.c_int, ip, ip, ip, C.c_int, dp, dp, dp, ip, C.c_int]
        L.or_energy.argtypes = [S, S, P, ip]
        L.or_energy.restype = C.c_double
        L.or_feasible.argtypes = [S, S, P, ip]
        L.or_brute.argtypes = [S, S, P, C.c_int, dp, ip, C.POINTER(C.c_longlong)]
        L.or_unary.argtypes = [S, C.c_int, S, C.c_int, C.c_double]
        L.or_unary.restype = C.c_double
        L.or_delta.argtypes = [C.c_double] * 4
        L.or_delta.restype = C.c_double
        L.or_angle.argtypes = [C.c_double] * 6
        L.or_angle.restype = C.c_double
        L.or_wrap.argtypes = [C.c_double]
        L.or_wrap.restype = C.c_double
        L.or_distortion.argtypes = [S, C.c_int, S, C.c_int, C.c_int, C.c_int, C.c_double]
        L.or_distortion.restype = C.c_double
        L.or_minnode_at.argtypes = [S, C.c_int, C.c_int]
        _lib = L
    return _lib


# ----------------------------------------------------------------- containers
@dataclass
class NodeSet:
    """Nodes in fp64 (model chain or frame-sorted scene / window)."""

    t: np.ndarray  # int32
    x: np.ndarray  # float64
    y: np.ndarray
    f: np.ndarray  # float64 [n, F]

    @property
    def n(self):
        return int(self.t.shape[0])

    def cstruct(self):
        keep = [np.ascontiguousarray(self.t, dtype=np.int32), np.ascontiguousarray(self.x, np.float64),
                np.ascontiguousarray(self.y, np.float64), np.ascontiguousarray(self.f, np.float64)]
        t, x, y, f = keep
        st = _Set(self.n, int(f.shape[1]) if f.ndim == 2 else 1, t.ctypes.data_as(C.POINTER(C.c_int)),
                  x.ctypes.data_as(C.POINTER(C.c_double)), y.ctypes.data_as(C.POINTER(C.c_double)),
                  f.ctypes.data_as(C.POINTER(C.c_double)))
        st._keep = keep  # the struct owns its arrays (no dangling pointers)
        return st

    def slice(self, lo, hi):
        return NodeSet(self.t[lo:hi], self.x[lo:hi], self.y[lo:hi], self.f[lo:hi])


def _params(p: dict) -> _Params:
    return _Params(float(p.get("lambda1", 0.6)), float(p.get("lambda2", 0.2)), float(p.get("lambda3", 5.0)),
                   float(p.get("w_dummy", 1.0)), int(p.get("T", 10)))


# --------------------------------------------------------- graph construction
def model_chain(frame, saliency) -> np.ndarray:
    """PAPER.md L198 (§2.1): "keeping only a single interest point per model frame
    ... choosing the most salient one"; empty frames have no node (L200).
    Saliency ties keep the earliest input point (D-1).  Returns input
    indices ordered by frame."""
    frame = np.asarray(frame)
    saliency = np.asarray(saliency)
    best = {}
    for k in range(frame.shape[0]):  # plain scan in input order
        f = int(frame[k])
        if f not in best or saliency[k] > saliency[best[f]]:
            best[f] = k
    return np.array([best[f] for f in sorted(best)], dtype=np.int64)


def model_chain_rank(frame, saliency, rank: int) -> np.ndarray:
    """Chain `rank` of the independent-chains model ("Multiple
    points 2: creation of several single point models (several second order
    chains)"): per occupied frame the point of saliency rank `rank` (0 = most
    salient = model_chain; ties: earlier input point ranks first, D-1); frames with
    <= rank points have no node.  Returns input indices ordered by frame."""
    frame = np.asarray(frame)
    saliency = np.asarray(saliency)
    per = {}
    for k in range(frame.shape[0]):  # plain scan in input order
        per.setdefault(int(frame[k]), []).append(k)
    out = []
    for f in sorted(per):
        ranked = sorted(per[f], key=lambda k: (-float(saliency[k]), k))
        if rank < len(ranked):
            out.append(ranked[rank])
    return np.array(out, dtype=np.int64)


def model_nodes_rank(pts, rank: int) -> NodeSet:
    idx = model_chain_rank(pts.frame, pts.saliency, rank)
    return NodeSet(pts.frame[idx].astype(np.int32), pts.x[idx].astype(np.float64),
                   pts.y[idx].astype(np.float64), pts.feat[idx].astype(np.float64))


def model_nodes(pts) -> NodeSet:
    idx = model_chain(pts.frame, pts.saliency)
    return NodeSet(pts.frame[idx].astype(np.int32), pts.x[idx].astype(np.float64),
                   pts.y[idx].astype(np.float64), pts.feat[idx].astype(np.float64))


def scene_sorted(frame) -> np.ndarray:
    """"assuming that the scene nodes are sorted in temporal (i.e.
    frame) order"; stable, so same-frame points keep input order."""
    return np.argsort(np.asarray(frame), kind="stable")


def scene_nodes(pts):
    order = scene_sorted(pts.frame)
    return order, NodeSet(pts.frame[order].astype(np.int32), pts.x[order].astype(np.float64),
                          pts.y[order].astype(np.float64), pts.feat[order].astype(np.float64))


def window_range(sorted_frames, o: int, W: int):
    """Block [o, o+W) of scene frames (A13): nodes with o <= t' < o+W."""
    t = np.asarray(sorted_frames)
    wb = int(np.count_nonzero(t < o))
    we = int(np.count_nonzero(t < o + W))
    return wb, we


# -------------------------------------------------------------------- solvers
def match(model: NodeSet, window: NodeSet, params: dict):
    """Exact minimiser for one (model, window): (E_dp, E_recomputed, A, z) with
    z[i] in 0..S-1 (window-local) or -1 for the dummy."""
    L = lib()
    m, s = model.cstruct(), window.cstruct()
    p = _params(params)
    E, Er, A = C.c_double(), C.c_double(), C.c_double()
    z = np.full(max(model.n, 1), -1, dtype=np.int32)
    L.or_match(C.byref(m), C.byref(s), C.byref(p), C.byref(E), C.byref(Er), C.byref(A),
               z.ctypes.data_as(C.POINTER(C.c_int)))
    return E.value, Er.value, A.value, z[: model.n].copy()


def match_batch(models: list[NodeSet], scene: NodeSet, params: dict, job_model, job_wb, job_we,
                n_threads: int | None = None):
    """Independent jobs (model index, window [wb, we)) over one sorted scene.
    z is reported as scene-sorted node index, -1 = dummy."""
    L = lib()
    n_threads = n_threads or os.cpu_count() or 1
    structs = [m.cstruct() for m in models]  # keeps the arrays alive for the call
    ms = (_Set * len(models))(*structs)
    s = scene.cstruct()
    p = _params(params)
    jm = np.ascontiguousarray(job_model, dtype=np.int32)
    jb = np.ascontiguousarray(job_wb, dtype=np.int32)
    je = np.ascontiguousarray(job_we, dtype=np.int32)
    n = int(jm.shape[0])
    Mmax = max(m.n for m in models)
    E = np.zeros(n)
    Er = np.zeros(n)
    A = np.zeros(n)
    z = np.full((n, Mmax), -1, dtype=np.int32)
    ip = C.POINTER(C.c_int)
    dp = C.POINTER(C.c_double)
    L.or_match_batch(ms, C.byref(s), C.byref(p), n, jm.ctypes.data_as(ip), jb.ctypes.data_as(ip),
                     je.ctypes.data_as(ip), int(n_threads), E.ctypes.data_as(dp), Er.ctypes.data_as(dp),
                     A.ctypes.data_as(dp), z.ctypes.data_as(ip), Mmax)
    return E, Er, A, z


def energy(model: NodeSet, window: NodeSet, params: dict, z) -> float:
    L = lib()
    zz = np.ascontiguousarray(z, dtype=np.int32)
    m, s = model.cstruct(), window.cstruct()
    p = _params(params)
    return L.or_energy(C.byref(m), C.byref(s), C.byref(p), zz.ctypes.data_as(C.POINTER(C.c_int)))


def feasible(model: NodeSet, window: NodeSet, params: dict, z) -> bool:
    L = lib()
    zz = np.ascontiguousarray(z, dtype=np.int32)
    m, s = model.cstruct(), window.cstruct()
    p = _params(params)
    return bool(L.or_feasible(C.byref(m), C.byref(s), C.byref(p), zz.ctypes.data_as(C.POINTER(C.c_int))))


def brute(model: NodeSet, window: NodeSet, params: dict, prune: bool = True):
    """DFS over the feasible set (hgm_brute.c): (E, z, n_leaves)."""
    L = lib()
    m, s = model.cstruct(), window.cstruct()
    p = _params(params)
    E = C.c_double()
    n = C.c_longlong()
    z = np.full(max(model.n, 1), -1, dtype=np.int32)
    L.or_brute(C.byref(m), C.byref(s), C.byref(p), int(prune), C.byref(E),
               z.ctypes.data_as(C.POINTER(C.c_int)), C.byref(n))
    return E.value, z[: model.n].copy(), n.value


# --------------------------------------------------------------------- detect
@dataclass
class DetectResult:
    winner: np.ndarray  # int32 [n_off], -1 when above threshold
    score: np.ndarray  # float64 [n_off]
    E: np.ndarray  # float64 [n_models, n_off]  DP optimum
    E_re: np.ndarray  # energy of the returned assignment, recomputed
    A: np.ndarray  # appearance distance
    z: np.ndarray  # int64 [n_models, n_off, Mmax] caller point ids, -1 = dummy


def offsets_list(first_frame: int, stride: int, count: int) -> np.ndarray:
    return first_frame + stride * np.arange(count, dtype=np.int64)


def detect(models_pts, scene_pts, params: dict, first_frame: int, stride: int, count: int, window: int,
           score_mode: int = 0, threshold: float = float("inf"), pairs=None, n_threads=None) -> DetectResult:
    """Per-offset nearest-model detection (PAPER.md L712 NPC; A14): for every
    offset o, winner(o) = the smallest m attaining min_m score(m, o), score =
    E* (score_mode 0) or A (score_mode 1); -1 if the minimum exceeds threshold.
    `pairs` (optional list of (m, k)) restricts the oracle to a sample; then
    only E/A/z of those pairs are filled (NaN elsewhere) and winners are -2."""
    models = [model_nodes(m) for m in models_pts]
    order, scene = scene_nodes(scene_pts)
    ids = scene_pts.ids()[order]
    offs = offsets_list(first_frame, stride, count)
    rng = [window_range(scene.t, int(o), window) for o in offs]
    if pairs is None:
        pairs = [(m, k) for k in range(count) for m in range(len(models))]
    pairs = list(pairs)
    jm = np.array([p[0] for p in pairs], dtype=np.int32)
    jb = np.array([rng[p[1]][0] for p in pairs], dtype=np.int32)
    je = np.array([rng[p[1]][1] for p in pairs], dtype=np.int32)
    E, Er, A, z = match_batch(models, scene, params, jm, jb, je, n_threads)
    nm = len(models)
    Mmax = max(m.n for m in models)
    EE = np.full((nm, count), np.nan)
    ER = np.full((nm, count), np.nan)
    AA = np.full((nm, count), np.nan)
    ZZ = np.full((nm, count, Mmax), -1, dtype=np.int64)
    for j, (m, k) in enumerate(pairs):
        EE[m, k], ER[m, k], AA[m, k] = E[j], Er[j], A[j]
        zz = z[j, : models[m].n]
        ZZ[m, k, : models[m].n] = np.where(zz >= 0, ids[np.maximum(zz, 0)], -1)
    S = EE if score_mode == 0 else AA
    winner = np.full(count, -2, dtype=np.int32)
    score = np.full(count, np.nan)
    for k in range(count):
        col = S[:, k]
        if np.all(np.isfinite(col)):
            w = int(np.argmin(col))  # first minimum = lowest model index (D-12)
            winner[k] = w if col[w] <= threshold else -1
            score[k] = col[w]
    return DetectResult(winner, score, EE, ER, AA, ZZ)


# ----------------------------------------------------------------- recognition
@dataclass
class ClassifyResult:
    block_label: np.ndarray  # int32 [n_blocks], -1 = no prototype within threshold
    block_score: np.ndarray  # float64 [n_blocks]: appearance distance of the nearest prototype
    block_proto: np.ndarray  # int32 [n_blocks]: index of the nearest prototype (-1 as above)
    clip_label: int  # majority vote over labelled blocks, ties -> smallest label; -1 if none
    A: np.ndarray  # float64 [n_prototypes, n_blocks]


def majority_vote(labels) -> int:
    """SPEC 'per-block classification aggregates to a stream label by majority
    vote over blocks' (reading R-f1b: ties -> smallest label;
    unlabelled blocks (-1) abstain; no labelled block -> -1)."""
    counts = {}
    for l in labels:
        l = int(l)
        if l >= 0:
            counts[l] = counts.get(l, 0) + 1
    if not counts:
        return -1
    top = max(counts.values())
    return min(l for l, c in counts.items() if c == top)


def classify_blocks(prototypes_pts, labels, scene_pts, params: dict, first_frame: int, stride: int, count: int,
                    window: int, threshold: float = float("inf"), n_threads=None) -> ClassifyResult:
    """Nearest prototype classifier (Sec. 4): every prototype is
    matched against every scene block (block k = frames [first_frame + k*stride,
    + window), L739-743 '60 frames'), the distance is the appearance part A of the
    optimal assignment ('only the appearance terms U(.) are used', L712), the block
    takes the label of the nearest prototype (lowest index on ties, D-12) and the
    clip label is the majority vote over blocks (SPEC)."""
    r = detect(prototypes_pts, scene_pts, params, first_frame, stride, count, window, score_mode=1,
               threshold=threshold, n_threads=n_threads)
    labels = np.asarray(labels, dtype=np.int32)
    bl = np.where(r.winner >= 0, labels[np.maximum(r.winner, 0)], -1).astype(np.int32)
    return ClassifyResult(bl, r.score, r.winner, majority_vote(bl), r.A)


# ------------------------------------------------------- independent chains
def chain_points(pts, rank: int):
    """The raw points of chain `rank` as a point set of the same type (so that
    detect() can take it as a model): rank-r selection, then model_chain of it is
    the identity (one point per frame)."""
    return pts.take(model_chain_rank(pts.frame, pts.saliency, rank))


def detect_chains(models_pts, n_chains: int, scene_pts, params: dict, first_frame: int, stride: int, count: int,
                  window: int, score_mode: int = 0, threshold: float = float("inf"), n_threads=None):
    """PAPER.md L756-761 "Multiple points 2": each model becomes up to n_chains single
    point chains (chain_points, ranks no frame reaches dropped), every chain is matched
    independently, and a model's distance is the average over its chains; then the
    per-offset nearest model (D-12 ties).  Returns (winner, score, S [n_models, count],
    chain_model)."""
    chains, chain_model = [], []
    for m, pts in enumerate(models_pts):
        for r in range(n_chains):
            idx = model_chain_rank(pts.frame, pts.saliency, r)
            if idx.size == 0:
                break
            chains.append(pts.take(idx))
            chain_model.append(m)
    r = detect(chains, scene_pts, params, first_frame, stride, count, window, score_mode=score_mode,
               n_threads=n_threads)
    Sc = r.E if score_mode == 0 else r.A
    cm = np.array(chain_model)
    S = np.stack([Sc[cm == m].mean(axis=0) for m in range(len(models_pts))])
    winner = np.full(count, -1, dtype=np.int32)
    score = np.full(count, np.nan)
    for k in range(count):
        w = int(np.argmin(S[:, k]))
        winner[k] = w if S[w, k] <= threshold else -1
        score[k] = S[w, k]
    return winner, score, S, cm
