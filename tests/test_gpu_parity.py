"""GPU parity: libhgm.so (through the C ABI) against the fp64 CPU oracle on the
same seeded inputs.  Marked gpu: runs on a B200 only."""
import math

import numpy as np
import pytest

import oracle
import synth
from tests._parity import Checker, tol

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def hgm():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1505_00581_b200 import hgm as H

    H.lib()
    return H


def _run_and_check(H, wl, scene_idx=0, ks=None, max_ties=0.01, models=None):
    p = wl.params()
    scene_pts = wl.scenes[scene_idx]
    count = wl.count[scene_idx]
    chk = Checker(wl.models, scene_pts, p, wl.first[scene_idx], wl.stride, wl.window)
    scene = H.build_scene_index(scene_pts, device=0, T_max=p["T"])
    mids = range(len(wl.models)) if models is None else models
    ks = list(range(count)) if ks is None else list(ks)
    pairs = [(m, k) for m in mids for k in ks]
    E_o, _, A_o, z_o = chk.oracle_pairs(pairs)
    gpu = {}
    for m in mids:
        mh = H.build_model_graph(wl.models[m], device=0)
        r = H.match_model_at_offsets(mh, scene, p, wl.first[scene_idx], wl.stride, count, wl.window,
                                     device_out=False)
        gpu[m] = r
    bad, ties = [], 0
    for j, (m, k) in enumerate(pairs):
        r = gpu[m]
        msg = chk.check_pair(m, k, r.E[k], r.A[k], r.z[k], E_o[j], A_o[j], z_o[j])
        if msg == "TIE":
            ties += 1
        elif msg:
            bad.append(msg)
    assert not bad, bad[:5]
    assert ties <= max(1, max_ties * len(pairs)), f"{ties} near-ties of {len(pairs)}"
    return len(pairs), ties


@pytest.mark.parametrize("block", range(5))
def test_c0_seeds(hgm, block):
    """C0 tiny (M=8, ~40 points, T=5): 200 seeds per block."""
    for seed in range(block * 200, block * 200 + 200):
        wl = synth.make_workload("C0", seed=seed)
        _run_and_check(hgm, wl, max_ties=1.0)


def test_c0_T10(hgm):
    for seed in range(100):
        wl = synth.make_workload("C0", seed=seed, T=10)
        _run_and_check(hgm, wl, max_ties=1.0)


def test_c1_all_offsets(hgm):
    """C1: one M=30 model against a 600-frame clip, all 541 offsets."""
    n, ties = _run_and_check(hgm, synth.make_workload("C1"))
    assert n == 541


def test_c2_sampled(hgm):
    wl = synth.make_workload("C2")
    rng = np.random.default_rng(2)
    for clip in rng.choice(25, 3, replace=False):
        ks = np.sort(rng.choice(wl.count[clip], 40, replace=False))
        _run_and_check(hgm, wl, scene_idx=int(clip), ks=ks)


def test_c3_sampled_short(hgm):
    wl = synth.make_workload("C3", n_frames=3000)
    rng = np.random.default_rng(3)
    ks = np.sort(rng.choice(wl.count[0], 60, replace=False))
    _run_and_check(hgm, wl, ks=ks)


def test_c4_sampled(hgm):
    wl = synth.make_workload("C4", T=10, n_frames=1200)
    _run_and_check(hgm, wl, ks=[0, 40], models=[0, 3])


def test_detect_matches_oracle(hgm):
    """detect_actions winners bit-exact against the oracle (ties: near-tie rule)."""
    wl = synth.make_workload("C2")
    clip = 4
    p = wl.params()
    count = 120
    ref = oracle.detect(wl.models, wl.scenes[clip], p, 0, 1, count, wl.window)
    scene = hgm.build_scene_index(wl.scenes[clip], device=0, T_max=10)
    models = [hgm.build_model_graph(m, device=0) for m in wl.models]
    det = hgm.detect_actions(models, scene, p, 0, 1, count, wl.window, want_E_all=True, device_out=False)
    for k in range(count):
        E_ref = ref.E[:, k]
        assert np.all(np.abs(det.E_all[:, k] - E_ref) <= 1e-6 + 1e-5 * np.abs(E_ref)), k
        w = int(det.winner[k])
        if w != int(ref.winner[k]):  # accept only a near-tie between the two winners
            assert abs(E_ref[w] - E_ref[ref.winner[k]]) <= tol(E_ref[ref.winner[k]]), k
        assert abs(float(det.score[k]) - ref.score[k]) <= tol(ref.score[k])


def test_detect_appearance_score_and_threshold(hgm):
    wl = synth.make_workload("C1")
    p = wl.params()
    scene = hgm.build_scene_index(wl.scenes[0], device=0, T_max=10)
    models = [hgm.build_model_graph(wl.models[0], device=0)]
    r = hgm.match_model_at_offsets(models[0], scene, p, 0, 1, 50, 60, device_out=False)
    det = hgm.detect_actions(models, scene, p, 0, 1, 50, 60, score_mode=1, threshold=float(np.median(r.A)),
                             device_out=False)
    assert np.array_equal(det.score, r.A)
    assert np.array_equal(det.winner, np.where(r.A > np.median(r.A), -1, 0))


def test_edge_cases(hgm):
    """Windows past the end, empty windows, M=1, M=2, T=1, coincident points."""
    p = dict(lambda1=0.6, lambda2=0.2, lambda3=5.0, w_dummy=1.0, T=5)
    rng = np.random.default_rng(7)
    for M in (1, 2, 3):
        wl = synth.make_workload("C0", seed=M)
        model_pts = wl.models[0].take(np.arange(M))
        scene_pts = wl.scenes[0]
        chk = Checker([model_pts], scene_pts, p, -10, 3, 8)
        scene = hgm.build_scene_index(scene_pts, device=0, T_max=5)
        mh = hgm.build_model_graph(model_pts, device=0)
        count = 15  # windows from frame -10 to past the last frame (20)
        r = hgm.match_model_at_offsets(mh, scene, p, -10, 3, count, 8, device_out=False)
        pairs = [(0, k) for k in range(count)]
        E_o, _, A_o, z_o = chk.oracle_pairs(pairs)
        for j, (m, k) in enumerate(pairs):
            msg = chk.check_pair(m, k, r.E[k], r.A[k], r.z[k], E_o[j], A_o[j], z_o[j])
            assert msg in (None, "TIE"), msg
        # empty windows: all dummies, E = lambda1 M W^d
        assert math.isclose(float(r.E[0]), 0.6 * M * 1.0, rel_tol=1e-6)
        assert list(r.z[0]) == [-1] * M
    # coincident points and T = 1
    pts = synth.gen_clutter(12, 0, 3.0, 4, rng)
    pts.x[:] = np.round(pts.x / 40) * 40  # many spatial coincidences
    pts.y[:] = np.round(pts.y / 40) * 40
    model_pts = synth.gen_model(1, 6, 1, 4, "edge", 0, gap2_prob=0.0)
    model_pts.x[:] = np.round(model_pts.x / 40) * 40
    model_pts.y[:] = np.round(model_pts.y / 40) * 40
    for T in (1, 2, 4):
        pp = dict(p, T=T)
        chk = Checker([model_pts], pts, pp, 0, 1, 12)
        scene = hgm.build_scene_index(pts, device=0, T_max=4)
        mh = hgm.build_model_graph(model_pts, device=0)
        r = hgm.match_model_at_offsets(mh, scene, pp, 0, 1, 1, 12, device_out=False)
        E_o, _, A_o, z_o = chk.oracle_pairs([(0, 0)])
        msg = chk.check_pair(0, 0, r.E[0], r.A[0], r.z[0], E_o[0], A_o[0], z_o[0])
        assert msg in (None, "TIE"), msg


def test_errors(hgm):
    wl = synth.make_workload("C0", seed=0)
    scene = hgm.build_scene_index(wl.scenes[0], device=0, T_max=5)
    model = hgm.build_model_graph(wl.models[0], device=0)
    with pytest.raises(hgm.HGMError) as e:
        hgm.match_model_at_offsets(model, scene, dict(T=6), 0, 1, 1, 20)
    assert e.value.status == 3  # T > T_max
    with pytest.raises(hgm.HGMError) as e:
        hgm.match_model_at_offsets(model, scene, dict(lambda1=-1.0, T=5), 0, 1, 1, 20)
    assert e.value.status == 3
    with pytest.raises(hgm.HGMError) as e:
        hgm.detect_actions([], scene, dict(T=5), 0, 1, 1, 20)
    assert e.value.status == 1
    other = synth.make_workload("C1")
    m2 = hgm.build_model_graph(other.models[0], device=0)  # F = 162 vs scene F = 8
    with pytest.raises(hgm.HGMError) as e:
        hgm.detect_actions([m2], scene, dict(T=5), 0, 1, 1, 20)
    assert e.value.status == 2


def test_device_builders_match_host_builders(hgm):
    import torch

    wl = synth.make_workload("C1")
    p = wl.params()
    s_h = hgm.build_scene_index(wl.scenes[0], device=0, T_max=10)
    m_h = hgm.build_model_graph(wl.models[0], device=0)
    s_d = hgm.build_scene_index(hgm.DevicePoints.from_host(wl.scenes[0]), T_max=10)
    m_d = hgm.build_model_graph(hgm.DevicePoints.from_host(wl.models[0]))
    a = hgm.match_model_at_offsets(m_h, s_h, p, 0, 1, 100, 60)
    b = hgm.match_model_at_offsets(m_d, s_d, p, 0, 1, 100, 60)
    torch.cuda.synchronize()
    assert torch.equal(a.E, b.E) and torch.equal(a.z, b.z)


@pytest.mark.parametrize("name,kw", [("C1", {}), ("C2", {}), ("C3", dict(n_frames=1500)), ("C0", dict(seed=3))])
def test_tiled_kernel_bitexact_to_reference_kernel(hgm, name, kw, monkeypatch):
    """K-DP v1 (tiled, shared memory) and K-DP v0 (one thread per state) run the
    same per-candidate arithmetic (hgm_device.cuh): results must be bit-identical."""
    import torch

    wl = synth.make_workload(name, **kw)
    p = wl.params()
    s = hgm.build_scene_index(wl.scenes[0], device=0, T_max=p["T"])
    out = {}
    for kern in ("v0", "v1"):
        monkeypatch.setenv("HGM_KERNEL", kern)
        res = []
        for mp in wl.models:
            m = hgm.build_model_graph(mp, device=0)
            res.append(hgm.match_model_at_offsets(m, s, p, wl.first[0], wl.stride, wl.count[0], wl.window))
        torch.cuda.synchronize()
        out[kern] = res
    for a, b in zip(out["v0"], out["v1"]):
        assert torch.equal(a.E, b.E) and torch.equal(a.A, b.A) and torch.equal(a.z, b.z)


@pytest.mark.parametrize("name,kw", [("C2", {}), ("C3", dict(n_frames=2000)), ("C4", dict(T=10, n_frames=900)),
                                     ("C4", dict(T=20, n_frames=460)), ("C4", dict(T=40, n_frames=450)),
                                     ("C4", dict(T=80, n_frames=420))])
def test_model_batched_kernel_bitexact(hgm, name, kw, monkeypatch):
    """detect_actions batches the 6 models of equal M into one K-DP pass; the
    per-model reference kernels (HGM_KERNEL=v0) must give identical bits."""
    import torch

    wl = synth.make_workload(name, **kw)
    p = wl.params()
    s = hgm.build_scene_index(wl.scenes[0], device=0, T_max=p["T"])
    models = [hgm.build_model_graph(m, device=0) for m in wl.models]
    res = {}
    for kern in ("v0", "v1"):
        monkeypatch.setenv("HGM_KERNEL", kern)
        for mode in (0, 1):
            r = hgm.detect_actions(models, s, p, wl.first[0], wl.stride, wl.count[0], wl.window, score_mode=mode,
                                   want_E_all=True)
            torch.cuda.synchronize()
            res[(kern, mode)] = r
    for mode in (0, 1):
        a, b = res[("v0", mode)], res[("v1", mode)]
        assert torch.equal(a.E_all, b.E_all) and torch.equal(a.winner, b.winner) and torch.equal(a.score, b.score)


def test_dense_fallbacks_bitexact(hgm, monkeypatch):
    """Shared memory capped so that no tiling fits: detect_actions retries its 6-model
    batch one model at a time and each model falls back to the reference (v0) kernels;
    with a cap that only fits one model, the single-model tiled path runs.  Both must
    give the bits of the v0 kernels."""
    import torch

    wl = synth.make_workload("C2")
    p = wl.params()
    s = hgm.build_scene_index(wl.scenes[1], device=0, T_max=10)
    models = [hgm.build_model_graph(m, device=0) for m in wl.models]
    monkeypatch.setenv("HGM_KERNEL", "v0")
    ref = hgm.detect_actions(models, s, p, 0, 1, 80, wl.window, want_E_all=True)
    monkeypatch.setenv("HGM_KERNEL", "v1")
    for cap in ("4", "40", "64"):
        monkeypatch.setenv("HGM_SMEM_MAX_KB", cap)
        got = hgm.detect_actions(models, s, p, 0, 1, 80, wl.window, want_E_all=True)
        torch.cuda.synchronize()
        assert torch.equal(ref.E_all, got.E_all) and torch.equal(ref.winner, got.winner), cap


@pytest.mark.parametrize("smem_kb", [20, 32, 48, 110])
def test_tile_sizes_bitexact(hgm, smem_kb, monkeypatch):
    """Shared-memory budgets from tiny (one-frame tiles whose a-frames are split into
    chunks, single-stage items) to the default: every tiling gives the v0 bits."""
    import torch

    wl = synth.make_workload("C1")
    p = wl.params()
    s = hgm.build_scene_index(wl.scenes[0], device=0, T_max=10)
    m = hgm.build_model_graph(wl.models[0], device=0)
    monkeypatch.setenv("HGM_KERNEL", "v0")
    a = hgm.match_model_at_offsets(m, s, p, 0, 1, 541, 60)
    monkeypatch.setenv("HGM_KERNEL", "v1")
    monkeypatch.setenv("HGM_SMEM_KB", str(smem_kb))
    b = hgm.match_model_at_offsets(m, s, p, 0, 1, 541, 60)
    torch.cuda.synchronize()
    assert torch.equal(a.E, b.E) and torch.equal(a.z, b.z)


def test_bit_determinism(hgm):
    import torch

    wl = synth.make_workload("C1")
    p = wl.params()
    s = hgm.build_scene_index(wl.scenes[0], device=0, T_max=10)
    m = hgm.build_model_graph(wl.models[0], device=0)
    a = hgm.match_model_at_offsets(m, s, p, 0, 1, 541, 60)
    b = hgm.match_model_at_offsets(m, s, p, 0, 1, 541, 60)
    torch.cuda.synchronize()
    assert torch.equal(a.E, b.E) and torch.equal(a.A, b.A) and torch.equal(a.z, b.z)


@pytest.mark.parametrize("seed,exact", [(0, False), (1, False), (2, True)])
def test_classify_blocks_matches_oracle(hgm, seed, exact):
    """Recognition layer (f1): per-block labels / distances and the clip vote against
    oracle.classify_blocks; 6 classes x 2 prototypes (M=30), 8 blocks of 60 frames."""
    rs = synth.make_recognition(seed, count=8, exact=exact)
    p = rs.params()
    ref = oracle.classify_blocks(rs.prototypes, rs.labels, rs.scene, p, 0, rs.stride, rs.count, rs.block)
    scene = hgm.build_scene_index(rs.scene, device=0, T_max=p["T"])
    protos = [hgm.build_model_graph(m, device=0) for m in rs.prototypes]
    got = hgm.classify_blocks(protos, rs.labels, scene, p, 0, rs.stride, rs.count, rs.block)
    for k in range(rs.count):
        assert abs(float(got.block_score[k]) - ref.block_score[k]) <= tol(ref.block_score[k]), k
        if got.block_label[k] != ref.block_label[k]:  # only a near-tie between the two nearest may differ
            a = ref.A[:, k]
            w = int(np.argmin(np.where(rs.labels == got.block_label[k], a, np.inf)))
            assert abs(a[w] - a[ref.block_proto[k]]) <= tol(a[ref.block_proto[k]]), k
    assert got.clip_label == oracle.majority_vote(got.block_label)
    if exact:
        assert np.array_equal(got.block_label, rs.truth) and np.all(got.block_score == 0)
    # the distances equal the appearance scores of detect_actions(score_mode=1)
    det = hgm.detect_actions(protos, scene, p, 0, rs.stride, rs.count, rs.block, score_mode=1, device_out=False)
    assert np.array_equal(det.score, got.block_score)
    assert np.array_equal(np.where(det.winner >= 0, rs.labels[np.maximum(det.winner, 0)], -1), got.block_label)


def test_classify_blocks_threshold_and_errors(hgm):
    rs = synth.make_recognition(5, count=6)
    p = rs.params()
    scene = hgm.build_scene_index(rs.scene, device=0, T_max=p["T"])
    protos = [hgm.build_model_graph(m, device=0) for m in rs.prototypes]
    full = hgm.classify_blocks(protos, rs.labels, scene, p, 0, rs.stride, rs.count, rs.block)
    thr = float(np.median(full.block_score))
    r = hgm.classify_blocks(protos, rs.labels, scene, p, 0, rs.stride, rs.count, rs.block, threshold=thr)
    assert np.array_equal(r.block_label, np.where(full.block_score <= thr, full.block_label, -1))
    assert r.clip_label == oracle.majority_vote(r.block_label)
    r = hgm.classify_blocks(protos, rs.labels, scene, p, 0, rs.stride, rs.count, rs.block, threshold=-1.0)
    assert np.all(r.block_label == -1) and r.clip_label == -1
    bad = rs.labels.copy()
    bad[0] = 6
    with pytest.raises(hgm.HGMError):
        hgm.classify_blocks(protos, bad, scene, p, 0, rs.stride, rs.count, rs.block, n_labels=6)


def _single_check(hgm, wl, T, oracle_ref=True):
    p = wl.params()
    p["T"] = T
    chk = Checker(wl.models, wl.scenes[0], p, 0, 1, wl.window)
    scene = hgm.build_scene_index(wl.scenes[0], device=0, T_max=T)
    m = hgm.build_model_graph(wl.models[0], device=0)
    r = hgm.match_model_at_offsets(m, scene, p, 0, 1, 1, wl.window, device_out=False)
    if oracle_ref:
        E_o, _, A_o, z_o = chk.oracle_pairs([(0, 0)])
        msg = chk.check_pair(0, 0, r.E[0], r.A[0], r.z[0], E_o[0], A_o[0], z_o[0])
        assert msg in (None, "TIE"), msg
    return r, chk


@pytest.mark.parametrize("T,plant", [(10, True), (10, False), (40, False), (80, True)])
def test_single_instance_754_nodes(hgm, T, plant):
    """f2: one M=30 model against a whole 754-node / 723-frame scene in one window
    (Table 3), against the oracle."""
    _single_check(hgm, synth.make_single(0 if plant else 1, plant=plant), T)


@pytest.mark.parametrize("seed,plant", [(0, True), (2, False)])
def test_single_instance_unpruned(hgm, seed, plant):
    """f2, T = +inf: a 160-frame scene with T above its span,
    against the oracle (its O(S^3 M) cost bounds the size)."""
    wl = synth.make_single(seed, n_frames=160, n_nodes=190, plant=plant)
    _single_check(hgm, wl, 161)


def test_single_instance_unpruned_full_size_properties(hgm):
    """T = +inf at the paper's full size (754 nodes): the GPU assignment is feasible, its
    fp64 energy (oracle.energy) equals the GPU E*, and E*(inf) <= E*(80) <= E*(10)."""
    wl = synth.make_single(1, plant=False)
    Es = []
    for T in (10, 80, 724):
        r, chk = _single_check(hgm, wl, T, oracle_ref=False)
        Es.append(float(r.E[0]))
        wb, we = chk.window_of(0)
        win = chk.scene.slice(wb, we)
        zl = np.array([-1 if v < 0 else chk.id2pos[int(v)] - wb for v in r.z[0]], np.int32)
        p = dict(chk.params)
        assert oracle.feasible(chk.models[0], win, p, zl)
        Ez = oracle.energy(chk.models[0], win, p, zl)
        assert abs(Ez - Es[-1]) <= tol(Ez), (T, Ez, Es[-1])
    assert Es[2] <= Es[1] + tol(Es[1]) and Es[1] <= Es[0] + tol(Es[0]), Es


@pytest.mark.parametrize("score_mode", [0, 1])
def test_detect_chains_matches_oracle(hgm, score_mode):
    """f3 independent chains: 6 models of 2 points per frame -> 2 chains each, a C2 clip,
    30 offsets; per-model mean scores and winners against oracle.detect_chains."""
    wl = synth.make_workload("C2")
    p = wl.params()
    clip, count, stride = 7, 30, 18
    w_o, s_o, S_o, cm_o = oracle.detect_chains(wl.models, 2, wl.scenes[clip], p, 0, stride, count, 60,
                                               score_mode=score_mode)
    scene = hgm.build_scene_index(wl.scenes[clip], device=0, T_max=10)
    chains, cm = [], []
    for m, pts in enumerate(wl.models):
        ch = hgm.build_model_chains(pts, 2, device=0)
        for r, c in enumerate(ch):
            assert c.M == len(oracle.model_chain_rank(pts.frame, pts.saliency, r))
        chains += ch
        cm += [m] * len(ch)
    assert cm == cm_o.tolist()
    det = hgm.detect_chains(chains, cm, len(wl.models), scene, p, 0, stride, count, 60, score_mode=score_mode,
                            want_S_all=True, device_out=False)
    assert np.all(np.abs(det.E_all - S_o) <= 2 * tol(S_o)), np.max(np.abs(det.E_all - S_o))
    for k in range(count):
        w = int(det.winner[k])
        if w != int(w_o[k]):
            assert abs(S_o[w, k] - S_o[w_o[k], k]) <= 2 * tol(S_o[w_o[k], k]), k
        assert abs(float(det.score[k]) - s_o[k]) <= 2 * tol(s_o[k])


def test_chain_builder_errors(hgm):
    wl = synth.make_workload("C1")
    ch = hgm.build_model_chains(wl.models[0], 5, device=0)
    assert len(ch) == 2  # C1's model has 2 points in every occupied frame
    scene = hgm.build_scene_index(wl.scenes[0], device=0, T_max=10)
    with pytest.raises(hgm.HGMError):  # chains not grouped by model
        hgm.detect_chains(ch, [1, 0], 2, scene, wl.params(), 0, 1, 4, 60)
    with pytest.raises(hgm.HGMError):  # model 1 has no chain
        hgm.detect_chains(ch, [0, 0], 2, scene, wl.params(), 0, 1, 4, 60)


@pytest.mark.parametrize("cfg,hop,stride", [("C1", 1, 1), ("C1", 7, 1), ("C1", 60, 5), ("C2", 250, 1),
                                            ("C2", 33, 3)])
def test_stream_equals_one_shot_detect(hgm, cfg, hop, stride):
    """f4 streaming: pushing the scene `hop` frames at a time reports every offset once,
    in order, bit-identical to one detect_actions call over the whole scene."""
    wl = synth.make_workload(cfg)
    sc_pts = wl.scenes[0]
    p = wl.params()
    nf = int(sc_pts.frame.max()) + 1
    count = (nf - 60) // stride + 1
    models = [hgm.build_model_graph(m, device=0) for m in wl.models]
    scene = hgm.build_scene_index(sc_pts, device=0, T_max=p["T"])
    ref = hgm.detect_actions(models, scene, p, 0, stride, count, 60, device_out=False)
    st = hgm.Stream(models, p, window=60, stride=stride)
    ws, ss, nxt = [], [], 0
    for f0 in range(0, nf, hop):
        n = min(hop, nf - f0)
        sel = np.nonzero((sc_pts.frame >= f0) & (sc_pts.frame < f0 + n))[0]
        first, w, s = st.push(sc_pts.take(sel), n)
        if len(w):
            assert first == nxt * stride
            nxt += len(w)
        ws.append(w)
        ss.append(s)
    w, s = np.concatenate(ws), np.concatenate(ss)
    assert len(w) == count
    assert np.array_equal(w, ref.winner) and np.array_equal(s, ref.score)
    if cfg == "C1" and hop == 7:  # and against the oracle on the first offsets
        r = oracle.detect(wl.models, sc_pts, p, 0, stride, 25, 60)
        assert np.all(np.abs(s[:25] - r.score) <= 1e-6 + 1e-5 * np.abs(r.score))


def test_stream_errors(hgm):
    wl = synth.make_workload("C1")
    models = [hgm.build_model_graph(wl.models[0], device=0)]
    st = hgm.Stream(models, wl.params(), window=60, stride=1)
    sc = wl.scenes[0]
    with pytest.raises(hgm.HGMError):  # frames beyond the pushed range
        st.push(sc.take(np.nonzero(sc.frame < 20)[0]), 10)
    first, w, s = st.push(None, 59)  # nothing complete yet
    assert len(w) == 0


@pytest.mark.parametrize("gap", [(0, 75), (200, 380)])
def test_stream_through_silent_stretches(hgm, gap):
    """f4: frames without any point (at the start, or a 180-frame silence) give windows
    with no node; the stream still equals one-shot detect on the same scene."""
    wl = synth.make_workload("C1")
    sc0 = wl.scenes[0]
    sc_pts = sc0.take(np.nonzero((sc0.frame < gap[0]) | (sc0.frame >= gap[1]))[0])
    p = wl.params()
    nf = 600
    count = nf - 60 + 1
    models = [hgm.build_model_graph(m, device=0) for m in wl.models]
    scene = hgm.build_scene_index(sc_pts, device=0, T_max=p["T"])
    ref = hgm.detect_actions(models, scene, p, 0, 1, count, 60, device_out=False)
    st = hgm.Stream(models, p, window=60, stride=1)
    ws, ss = [], []
    for f0 in range(0, nf, 25):
        sel = np.nonzero((sc_pts.frame >= f0) & (sc_pts.frame < f0 + 25))[0]
        _, w, s = st.push(sc_pts.take(sel), 25)
        ws.append(w)
        ss.append(s)
    w, s = np.concatenate(ws), np.concatenate(ss)
    assert np.array_equal(w, ref.winner) and np.array_equal(s, ref.score)
    r = oracle.detect(wl.models, sc_pts, p, 0, 1, count, 60, pairs=[(0, k) for k in range(gap[0], gap[1] - 60 + 1, 17)])
    for k in range(gap[0], gap[1] - 60 + 1, 17):  # empty windows: the all-dummy energy
        assert abs(s[k] - r.E[0, k]) <= 1e-6 + 1e-5 * abs(r.E[0, k])
