"""Multi-GPU driver: one process per GPU, the (model, offset) grid sharded over
ranks, one collective at the end.

Every (model, offset) DP is independent (PAPER.md L777 proposes batching models
and spreading the trellises over the hardware), so there is no exchange until
the final per-offset argmin over models.  The ranks form an R_off x R_mod grid:

  * offset axis: contiguous offset ranges, balanced by the predicted work of
    every offset (exact real-triple candidate counts from the frame histogram,
    work.py); each rank builds its own scene index over the frames its windows
    touch, [o_begin, o_end + W) (halo W-1 frames);
  * model axis (only when offsets < ranks x 148 SMs, e.g. C1, C4):
    contiguous model ranges balanced by chain length (work ~ M - 2).

Each rank computes its block with libhgm.so and packs per-offset keys
(score bits << 32 | global model index), which order exactly like (score, model)
because scores are >= 0.  The one collective is
  * R_mod == 1: an all_gather of the rank's keys (8 B per offset);
  * R_mod > 1 : an all_reduce(MIN) of a full-length key vector (int64 max where
    the rank has no block) -- the model-axis argmin and the offset gather in one,
    deterministic and bit-exact, ties to the lowest model index.

`compute` is injectable so that the host logic (partitioning, slicing, key
packing) is testable with gloo on CPU; the product path uses libhgm.so.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .work import count_work

SMS_PER_GPU = 148  # B200
KEY_NONE = np.iinfo(np.int64).max


@dataclass
class Shard:
    rank: int
    k_begin: int  # first offset index (global)
    k_end: int
    frame_lo: int  # scene frames this rank needs: [frame_lo, frame_hi)
    frame_hi: int
    m_begin: int = 0  # model range [m_begin, m_end) (None = all models)
    m_end: int | None = None


def offset_work(frames, first_frame: int, stride: int, count: int, window: int, T: int) -> np.ndarray:
    """Predicted work of every offset: its real-triple candidates (+1 so empty windows
    still count), exact, vectorised over offsets."""
    if count <= 0:
        return np.zeros(0, np.float64)
    if frames is None or len(frames) == 0:
        return np.ones(count, np.float64)
    return count_work(frames, first_frame, stride, count, window, T, per_offset=True).astype(np.float64) + 1.0


def balanced_cuts(weights, parts: int) -> list[int]:
    """Cut points 0 = c_0 <= ... <= c_parts = n of contiguous ranges with near-equal
    weight sums (prefix-sum quantiles)."""
    n = len(weights)
    if parts <= 1 or n == 0:
        return [0] + [n] * max(parts, 1)
    c = np.concatenate([[0.0], np.cumsum(np.asarray(weights, np.float64))])
    cuts = [int(np.searchsorted(c, c[-1] * r / parts, side="left")) for r in range(parts + 1)]
    cuts[0], cuts[-1] = 0, n
    for r in range(1, parts + 1):
        cuts[r] = min(max(cuts[r], cuts[r - 1]), n)
    return cuts


def grid_shape(world: int, count: int, n_models: int) -> tuple[int, int]:
    """(R_off, R_mod): the model axis is used only when the offsets alone cannot fill
    the ranks' SMs (count < world x 148) and there are several models; then R_mod is
    the divisor of `world` (<= n_models) with the smallest per-rank block
    ceil(n_models / R_mod) x ceil(count / R_off), ties to fewer model groups."""
    if world <= 1 or n_models <= 1 or count >= world * SMS_PER_GPU:
        return world, 1
    best = None
    for d in range(1, min(world, n_models) + 1):
        if world % d:
            continue
        load = -(-n_models // d) * -(-count // (world // d))
        if best is None or load < best[0]:
            best = (load, d)
    return world // best[1], best[1]


def shard_offsets(frames, first_frame: int, stride: int, count: int, window: int, T: int, world: int,
                  model_sizes=None) -> list[Shard]:
    """One Shard per rank.  Offsets: contiguous, balanced by predicted work (every
    count).  Models (model_sizes = chain lengths, optional): a second axis when
    grid_shape asks for it, balanced by M - 2."""
    n_models = len(model_sizes) if model_sizes is not None else 1
    r_off, r_mod = grid_shape(world, count, n_models)
    ks = balanced_cuts(offset_work(frames, first_frame, stride, count, window, T), r_off) if count > 0 \
        else [0] * (r_off + 1)
    if r_mod > 1:
        ms = balanced_cuts([max(int(M) - 2, 0) + 1 for M in model_sizes], r_mod)
    else:
        ms = [0, None]
    out = []
    for r in range(max(world, 1)):
        so, sm = r // r_mod, r % r_mod
        kb, ke = ks[so], ks[so + 1]
        flo = first_frame + kb * stride
        fhi = first_frame + max(ke - 1, kb) * stride + window
        out.append(Shard(r, kb, ke, flo, fhi, ms[sm], ms[sm + 1]))
    return out


def pack_keys(score: np.ndarray, winner: np.ndarray) -> np.ndarray:
    """(float bits << 32) | model index: orders like (score, model) for score >= 0."""
    bits = np.asarray(score, np.float32).view(np.uint32).astype(np.uint64)
    return ((bits << np.uint64(32)) | np.asarray(winner, np.int64).astype(np.uint64) & np.uint64(0xFFFFFFFF)).view(
        np.int64)


def unpack_keys(keys: np.ndarray):
    u = np.asarray(keys, np.int64).view(np.uint64)
    score = (u >> np.uint64(32)).astype(np.uint32).view(np.float32)
    w = (u & np.uint64(0xFFFFFFFF)).astype(np.uint32).view(np.int32)
    return score, w


def gpu_compute(models_pts, scene_pts, params, first_frame, stride, count, window, score_mode, threshold):
    """Per-rank compute on the local GPU through libhgm.so (no threshold here: the
    threshold applies to the global minimum after the collective)."""
    from . import hgm

    T = int(params.get("T", 10))
    dev = _local_device()
    scene = hgm.build_scene_index(scene_pts, device=dev, T_max=T)
    models = [hgm.build_model_graph(m, device=dev) for m in models_pts]
    r = hgm.detect_actions(models, scene, params, first_frame, stride, count, window, score_mode,
                           threshold=float("inf"), device_out=False)
    return np.asarray(r.score, np.float32), np.asarray(r.winner, np.int32)


def _local_device():
    import torch

    return torch.cuda.current_device() if torch.cuda.is_available() else 0


def _model_sizes(models_pts):
    return [int(np.unique(np.asarray(m.frame)).size) for m in models_pts]


def detect_actions_sharded(models_pts, scene_pts, params: dict, first_frame: int, stride: int, count: int,
                           window: int = 60, score_mode: int = 0, threshold: float = float("inf"), group=None,
                           compute=None, device=None):
    """All ranks return the full (winner, score) arrays for all `count` offsets.
    `scene_pts` is the full scene (each rank slices its frames) or a callable
    (frame_lo, frame_hi) -> points that generates / loads only that slice."""
    import torch
    import torch.distributed as dist

    compute = compute or gpu_compute
    world = dist.get_world_size(group) if group is not None or dist.is_initialized() else 1
    rank = dist.get_rank(group) if world > 1 else 0
    T = int(params.get("T", 10))
    frames_all = None if callable(scene_pts) else np.asarray(scene_pts.frame)
    shards = shard_offsets(frames_all, first_frame, stride, count, window, T, world,
                           model_sizes=_model_sizes(models_pts))
    sh = shards[rank]
    m_lo, m_hi = sh.m_begin, (len(models_pts) if sh.m_end is None else sh.m_end)
    if callable(scene_pts):
        local = scene_pts(sh.frame_lo, sh.frame_hi)
    else:
        sel = np.nonzero((scene_pts.frame >= sh.frame_lo) & (scene_pts.frame < sh.frame_hi))[0]
        local = scene_pts.take(sel) if hasattr(scene_pts, "take") else scene_pts
    n_local = sh.k_end - sh.k_begin
    if n_local > 0 and m_hi > m_lo:
        score, winner = compute(models_pts[m_lo:m_hi], local, params, first_frame + sh.k_begin * stride, stride,
                                n_local, window, score_mode, threshold)
        winner = np.asarray(winner, np.int32) + np.int32(m_lo)  # global model index
    else:
        score, winner = np.zeros(0, np.float32), np.zeros(0, np.int32)
    keys = pack_keys(score, winner)
    model_axis = any(s.m_end is not None for s in shards)
    if world > 1:
        dev = device or (torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl"
                         else torch.device("cpu"))
        if model_axis:  # the one collective: argmin over the model axis + gather of the offset axis
            buf = torch.full((count,), KEY_NONE, dtype=torch.int64, device=dev)
            buf[sh.k_begin:sh.k_end] = torch.from_numpy(keys).to(dev)
            dist.all_reduce(buf, op=dist.ReduceOp.MIN, group=group)
            keys = buf.cpu().numpy()
        else:  # the one collective: 8 B per offset
            maxn = max(s.k_end - s.k_begin for s in shards)
            buf = torch.full((maxn,), -1, dtype=torch.int64, device=dev)
            buf[:n_local] = torch.from_numpy(keys).to(dev)
            parts = [torch.empty_like(buf) for _ in range(world)]
            dist.all_gather(parts, buf, group=group)
            keys = np.concatenate([parts[s.rank][: s.k_end - s.k_begin].cpu().numpy() for s in shards])
    score, winner = unpack_keys(keys)
    winner = np.where(score > threshold, -1, winner).astype(np.int32)
    return winner, score
