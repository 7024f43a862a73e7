"""Host logic: the roofline work counter and the multi-rank sharding driver
(world_size 2 over gloo on CPU; the per-rank compute is injected)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle
import synth
from paper_1505_00581_b200.dist import (balanced_cuts, detect_actions_sharded, grid_shape, offset_work, pack_keys,
                                        shard_offsets, unpack_keys)
from paper_1505_00581_b200.work import count_work


def _brute_counts(frames, first, stride, count, W, T):
    t = np.sort(np.asarray(frames))
    rc = rs = es = ec = 0
    for k in range(count):
        o = first + k * stride
        win = [n for n in range(t.size) if o <= t[n] < o + W]
        es += 2 * len(win) + 1
        ec += len(win)
        for b in win:
            ec += 2 * sum(1 for c in win if t[b] < t[c] < t[b] + T)
            for a in win:
                if t[a] < t[b] < t[a] + T:
                    rs += 1
                    rc += sum(1 for c in win if t[b] < t[c] < t[a] + T)
    return rc, rs, es, ec


@pytest.mark.parametrize("seed", range(6))
def test_count_work_matches_enumeration(seed):
    rng = np.random.default_rng(seed)
    frames = rng.integers(0, 40, size=int(rng.integers(5, 60)))
    T = int(rng.integers(1, 8))
    W = int(rng.integers(1, 25))
    stride = int(rng.integers(1, 4))
    first = int(rng.integers(-5, 10))
    count = int(rng.integers(1, 12))
    w = count_work(frames, first, stride, count, W, T)
    assert (w.real_candidates, w.real_states, w.eps_states, w.eps_candidates) == _brute_counts(
        frames, first, stride, count, W, T)


def test_paper_work_item_count():
    """M=30, S=60 -> M S^2 = 108000 work-items (unpruned trellis)."""
    M, S = 30, 60
    assert M * S * S == 108000
    # and the pruned cross-section is ~S x T: one point per frame, T=10
    frames = np.arange(S)
    w = count_work(frames, 0, 1, 1, S, 10)
    assert w.real_states <= S * 10


def test_pack_keys_order():
    s = np.array([3.5, 0.0, 3.5, np.inf, 1e-30], np.float32)
    m = np.array([2, 5, 1, 0, 7], np.int32)
    k = pack_keys(s, m)
    order = np.argsort(k.view(np.uint64), kind="stable")
    assert list(order) == [1, 4, 2, 0, 3]  # by (score, model)
    s2, m2 = unpack_keys(k)
    assert np.array_equal(s2, s) and np.array_equal(m2, m)


def test_shards_cover_offsets_contiguously():
    wl = synth.make_workload("C1")
    for world in (1, 2, 3, 8):
        sh = shard_offsets(wl.scenes[0].frame, 0, 1, 541, 60, 10, world)
        assert sh[0].k_begin == 0 and sh[-1].k_end == 541
        for a, b in zip(sh, sh[1:]):
            assert a.k_end == b.k_begin


def test_shards_balanced_by_predicted_work():
    """Offset ranges are balanced by the exact per-offset candidate counts for every
    count (no uniform fallback), and the per-offset counts sum to the total."""
    wl = synth.make_workload("C3", n_frames=6000)
    fr = wl.scenes[0].frame
    count = wl.count[0]
    per = offset_work(fr, 0, 1, count, 60, 10)
    assert int((per - 1).sum()) == count_work(fr, 0, 1, count, 60, 10).real_candidates
    for world in (2, 3, 8):
        sh = shard_offsets(fr, 0, 1, count, 60, 10, world)
        loads = [per[s.k_begin:s.k_end].sum() for s in sh]
        assert max(loads) <= per.sum() / world + per.max() + 1e-9, (world, loads)
        assert all(s.m_end is None for s in sh)  # count >= world x 148: offsets only


def test_grid_shape_and_model_cuts():
    assert grid_shape(8, 24941, 6) == (8, 1)      # C3: offsets fill the SMs
    assert grid_shape(8, 361, 6) == (4, 2)        # C4: 361 offsets < 8 x 148: 3 models x 91 offsets
    assert grid_shape(4, 541, 1) == (4, 1)        # one model: nothing to split
    assert grid_shape(2, 100, 6) == (2, 1)        # equal blocks: keep 6-model batches
    assert grid_shape(4, 2, 5) == (2, 2)          # both axes
    assert grid_shape(2, 1, 50) == (1, 2)         # one window, 50 models (the paper's context)
    assert balanced_cuts([1, 1, 1, 1], 2) == [0, 2, 4]
    assert balanced_cuts([10, 1, 1, 1], 2) == [0, 1, 4]
    wl = synth.make_workload("C4", T=10)
    sh = shard_offsets(wl.scenes[0].frame, 0, 10, wl.count[0], 400, 10, 8, model_sizes=[200] * 6)
    assert {(s.m_begin, s.m_end) for s in sh} == {(0, 3), (3, 6)}
    assert sorted({(s.k_begin, s.k_end) for s in sh})[0][0] == 0


def _fake_compute(models_pts, scene_pts, params, first_frame, stride, count, window, score_mode, threshold):
    """A deterministic stand-in for the per-rank compute: score of (model, offset) is a
    function of the model's points and the offset's absolute first frame only, with
    frequent exact ties between models (the lowest index must win)."""
    offs = first_frame + stride * np.arange(count)
    S = np.stack([((offs * 7 + int(m.x.sum()) * 3) % 11).astype(np.float32) for m in models_pts])
    return S.min(axis=0), S.argmin(axis=0).astype(np.int32)


def _fake_worker(rank, world, port, count, out):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    wl = synth.make_workload("C1")
    models = [synth.gen_model(c, 30, 2, synth.F_KTH, "dist-fake", 0) for c in range(5)]
    w, s = detect_actions_sharded(models, wl.scenes[0], wl.params(), 3, 1, count, 60, compute=_fake_compute)
    out[rank] = (w.tolist(), s.tolist())
    dist.destroy_process_group()


@pytest.mark.parametrize("world,count", [(2, 1), (4, 2), (3, 2), (2, 40), (3, 500), (4, 541)])
def test_sharded_grid_equals_single_process_gloo(world, count):
    """Both axes (offset ranges, model ranges with all_reduce(MIN) of packed keys) and
    the offset-only all_gather path give exactly the single-process argmin."""
    ctx = mp.get_context("spawn")
    out = ctx.Manager().dict()
    port = _free_port()
    procs = [ctx.Process(target=_fake_worker, args=(r, world, port, count, out)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
        assert p.exitcode == 0
    wl = synth.make_workload("C1")
    models = [synth.gen_model(c, 30, 2, synth.F_KTH, "dist-fake", 0) for c in range(5)]
    s_ref, w_ref = _fake_compute(models, wl.scenes[0], None, 3, 1, count, 60, 0, None)
    for r in range(world):
        w, s = out[r]
        assert w == w_ref.tolist() and s == s_ref.tolist()


def _oracle_compute(models_pts, scene_pts, params, first_frame, stride, count, window, score_mode, threshold):
    r = oracle.detect(models_pts, scene_pts, params, first_frame, stride, count, window, score_mode=score_mode)
    return r.score.astype(np.float32), r.winner.astype(np.int32)


def _worker(rank, world, port, out):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    wl = synth.make_workload("C1")
    w, s = detect_actions_sharded(wl.models * 2, wl.scenes[0], wl.params(), 100, 1, 40, 60, compute=_oracle_compute)
    out[rank] = (w.tolist(), s.tolist())
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_sharded_detect_equals_single_process_gloo():
    """Sharding invariance: world 2 (gloo) gives bit-identical winners and scores
    to a single process over all offsets."""
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
        assert p.exitcode == 0
    wl = synth.make_workload("C1")
    ref = oracle.detect(wl.models * 2, wl.scenes[0], wl.params(), 100, 1, 40, 60)
    for r in range(2):
        w, s = out[r]
        assert w == ref.winner.tolist()
        assert np.array_equal(np.array(s, np.float32), ref.score.astype(np.float32))


def test_bench_gpus_flag_spawns_ranks():
    """`python bench.py --gpus 2` without a launcher re-executes itself under
    torch.distributed.run (127.0.0.1): exactly one JSON line (rank 0) with n_gpus = 2.
    Exercised through the reference arm, which runs on the host cores (no GPU here)."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--gpus", "2",
                          "--steps", "1", "--warmup", "0", "--cpu-seconds", "1", "--frames-per-gpu", "800"],
                         capture_output=True, text=True, timeout=300, env=env, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["impl"] == "reference" and d["value"] > 0
    assert "spawning 2 ranks" in out.stderr
