"""Host logic: the roofline work counter and the multi-rank sharding driver
(world_size 2 over gloo on CPU; the per-rank compute is injected)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle
import synth
from paper_1505_00581_b200.dist import detect_actions_sharded, pack_keys, shard_offsets, unpack_keys
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
