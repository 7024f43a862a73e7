"""Multi-GPU driver: one process per GPU, offsets sharded by contiguous ranges,
one collective at the end.

Every (model, offset) DP is independent (PAPER.md L777 proposes exactly this
batching), so there is no exchange until the final per-offset argmin.  Rank r
  1. takes a contiguous offset range, balanced by predicted work;
  2. builds its own scene index over the frames its windows touch
     [o_begin, o_end + W) (halo W-1 frames);
  3. runs detect_actions on its range;
  4. all_gathers packed per-offset keys (score bits << 32 | model) -- one
     collective of 8 bytes per offset (torch.distributed, NCCL over NVLink).

`compute` is injectable so that the host logic (partitioning, slicing,
gathering) is testable with gloo on CPU; the product path uses libhgm.so.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .work import count_work


@dataclass
class Shard:
    rank: int
    k_begin: int  # first offset index (global)
    k_end: int
    frame_lo: int  # scene frames this rank needs: [frame_lo, frame_hi)
    frame_hi: int


def shard_offsets(frames, first_frame: int, stride: int, count: int, window: int, T: int, world: int) -> list[Shard]:
    """Contiguous offset ranges with near-equal predicted candidate counts."""
    if world <= 1 or count <= 1:
        ks = [0, count]
    else:
        per = np.array([count_work(frames, first_frame + k * stride, stride, 1, window, T).real_candidates + 1
                        for k in range(count)], dtype=np.float64) if count <= 4096 else None
        if per is None:  # long scenes: per-offset work ~ uniform in expectation; split by count
            ks = [round(count * r / world) for r in range(world + 1)]
        else:
            c = np.concatenate([[0], np.cumsum(per)])
            ks = [int(np.searchsorted(c, c[-1] * r / world)) for r in range(world + 1)]
            ks[0], ks[-1] = 0, count
            for r in range(1, world + 1):
                ks[r] = max(ks[r], ks[r - 1])
    out = []
    for r in range(max(world, 1)):
        kb, ke = ks[r], ks[r + 1]
        flo = first_frame + kb * stride
        fhi = first_frame + max(ke - 1, kb) * stride + window
        out.append(Shard(r, kb, ke, flo, fhi))
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
    """Per-rank compute on the local GPU through libhgm.so."""
    from . import hgm

    T = int(params.get("T", 10))
    scene = hgm.build_scene_index(scene_pts, device=_local_device(), T_max=T)
    models = [hgm.build_model_graph(m, device=_local_device()) for m in models_pts]
    r = hgm.detect_actions(models, scene, params, first_frame, stride, count, window, score_mode,
                           threshold=float("inf"), device_out=False)
    return np.asarray(r.score, np.float32), np.asarray(r.winner, np.int32)


def _local_device():
    import torch

    return torch.cuda.current_device() if torch.cuda.is_available() else 0


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
    frames_all = None if callable(scene_pts) else scene_pts.frame
    shards = shard_offsets(frames_all if frames_all is not None else np.zeros(0, np.int64), first_frame, stride,
                           count, window, T, world) if frames_all is not None else \
        shard_offsets(np.zeros(0), first_frame, stride, count, window, T, world)
    sh = shards[rank]
    if callable(scene_pts):
        local = scene_pts(sh.frame_lo, sh.frame_hi)
    else:
        sel = np.nonzero((scene_pts.frame >= sh.frame_lo) & (scene_pts.frame < sh.frame_hi))[0]
        local = scene_pts.take(sel) if hasattr(scene_pts, "take") else scene_pts
    n_local = sh.k_end - sh.k_begin
    if n_local > 0:
        score, winner = compute(models_pts, local, params, first_frame + sh.k_begin * stride, stride, n_local, window,
                                score_mode, threshold)
    else:
        score, winner = np.zeros(0, np.float32), np.zeros(0, np.int32)
    keys = pack_keys(score, winner)
    if world > 1:
        maxn = max(s.k_end - s.k_begin for s in shards)
        dev = device or (torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl"
                         else torch.device("cpu"))
        buf = torch.full((maxn,), -1, dtype=torch.int64, device=dev)
        buf[:n_local] = torch.from_numpy(keys).to(dev)
        parts = [torch.empty_like(buf) for _ in range(world)]
        dist.all_gather(parts, buf, group=group)  # the one collective: 8 B per offset
        keys = np.concatenate([parts[s.rank][: s.k_end - s.k_begin].cpu().numpy() for s in shards])
    score, winner = unpack_keys(keys)
    winner = np.where(score > threshold, -1, winner).astype(np.int32)
    return winner, score
