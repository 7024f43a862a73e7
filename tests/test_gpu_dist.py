"""Multi-rank path with the product compute: 2 processes share cuda:0 over gloo, each
running its shard through libhgm.so (dist.gpu_compute), and the gathered result must be
bit-identical to one process's detect_actions over all offsets.
Covers the offset axis (all_gather) and the model axis (all_reduce(MIN) of packed keys)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import synth

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, clip, first, count, score_mode, out):
    import torch
    import torch.distributed as dist

    from paper_1505_00581_b200.dist import detect_actions_sharded, shard_offsets

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    wl = synth.make_workload("C2")
    sizes = [int(np.unique(m.frame).size) for m in wl.models]
    sh = shard_offsets(wl.scenes[clip].frame, first, 1, count, 60, 10, world, model_sizes=sizes)
    w, s = detect_actions_sharded(wl.models, wl.scenes[clip], wl.params(), first, 1, count, 60,
                                  score_mode=score_mode)
    out[rank] = (w.tolist(), np.asarray(s, np.float32).tolist(),
                 [(x.k_begin, x.k_end, x.m_begin, x.m_end) for x in sh])
    dist.destroy_process_group()


@pytest.mark.parametrize("count,score_mode,axis", [(300, 0, "offsets"), (3, 0, "models"), (1, 1, "models")])
def test_two_ranks_on_gpu_equal_one_process(count, score_mode, axis):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1505_00581_b200 import hgm

    clip, first = 5, 17
    ctx = mp.get_context("spawn")
    out = ctx.Manager().dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, clip, first, count, score_mode, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(600)
        assert p.exitcode == 0
    wl = synth.make_workload("C2")
    scene = hgm.build_scene_index(wl.scenes[clip], device=0, T_max=10)
    models = [hgm.build_model_graph(m, device=0) for m in wl.models]
    ref = hgm.detect_actions(models, scene, wl.params(), first, 1, count, 60, score_mode=score_mode,
                             device_out=False)
    for r in range(2):
        w, s, shards = out[r]
        if axis == "models":
            assert any(m_end is not None for _, _, _, m_end in shards), shards
        else:
            assert all(m_end is None for _, _, _, m_end in shards), shards
        assert w == np.asarray(ref.winner).tolist()
        assert np.array_equal(np.asarray(s, np.float32), np.asarray(ref.score, np.float32))
