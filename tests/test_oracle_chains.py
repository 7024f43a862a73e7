"""Oracle pins for the independent-chains model (PAPER.md L756-761
"Multiple points 2": several single point chains, solved independently, distance =
average over the chains)."""
import numpy as np
import pytest

import oracle
import synth


def test_rank_selection_hand_case():
    # frame 0: saliencies .5 .9 .5 (input 0, 1, 2); frame 3: .2; frame 1: .7 .7
    frame = np.array([0, 0, 3, 0, 1, 1])
    sal = np.array([.5, .9, .2, .5, .7, .7])
    assert oracle.model_chain_rank(frame, sal, 0).tolist() == [1, 4, 2]
    assert oracle.model_chain_rank(frame, sal, 1).tolist() == [0, 5]  # tie .5/.5 -> earlier input first
    assert oracle.model_chain_rank(frame, sal, 2).tolist() == [3]
    assert oracle.model_chain_rank(frame, sal, 3).tolist() == []


@pytest.mark.parametrize("seed", range(20))
def test_chains_partition_the_points(seed):
    """Chains 0..K-1 (K = the largest per-frame count) use every point exactly once;
    chain r has a node in exactly the frames holding more than r points; chain 0 is
    the paper's single-point chain (L198); saliency is non-increasing with the rank."""
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 40))
    frame = rng.integers(0, 10, n)
    sal = rng.integers(0, 4, n) / 4.0  # many ties
    K = np.bincount(frame).max()
    used = np.concatenate([oracle.model_chain_rank(frame, sal, r) for r in range(K)])
    assert sorted(used.tolist()) == list(range(n))
    assert oracle.model_chain_rank(frame, sal, 0).tolist() == oracle.model_chain(frame, sal).tolist()
    cnt = np.bincount(frame, minlength=10)
    for r in range(K):
        idx = oracle.model_chain_rank(frame, sal, r)
        assert frame[idx].tolist() == [f for f in range(10) if cnt[f] > r]
        if r:
            prev = dict(zip(frame[oracle.model_chain_rank(frame, sal, r - 1)].tolist(),
                            sal[oracle.model_chain_rank(frame, sal, r - 1)].tolist()))
            assert all(sal[k] <= prev[int(frame[k])] for k in idx)


def _set():
    wl = synth.make_workload("C1", n_frames=120)
    models = [wl.models[0], synth.gen_model(1, 30, 2, synth.F_KTH, "chains", 0)]
    return wl, models


def test_one_chain_equals_detect():
    wl, models = _set()
    p = wl.params()
    w, s, S, cm = oracle.detect_chains(models, 1, wl.scenes[0], p, 0, 5, 8, 60)
    r = oracle.detect(models, wl.scenes[0], p, 0, 5, 8, 60)
    assert np.array_equal(w, r.winner) and np.array_equal(S, r.E) and cm.tolist() == [0, 1]


def test_distance_is_the_mean_of_independent_chain_matches():
    """Against the definition: each chain matched alone by the DFS-verified single
    window oracle.match, then averaged."""
    wl, models = _set()
    p = wl.params()
    w, s, S, cm = oracle.detect_chains(models, 2, wl.scenes[0], p, 0, 7, 3, 60, score_mode=1)
    order, scene = oracle.scene_nodes(wl.scenes[0])
    for m in range(2):
        for k in range(3):
            wb, we = oracle.window_range(scene.t, 7 * k, 60)
            A = [oracle.match(oracle.model_nodes_rank(models[m], r), scene.slice(wb, we), p)[2] for r in range(2)]
            assert abs(S[m, k] - (A[0] + A[1]) / 2) <= 1e-12 * max(1.0, abs(S[m, k]))
    assert np.array_equal(w, np.argmin(S, axis=0))


def test_identical_chains_average_to_one_chain():
    """Two points per frame with equal geometry and descriptor (saliency differs):
    both chains are the same graph, so the average equals the single-chain distance."""
    wl, _ = _set()
    m = wl.models[0]
    k = oracle.model_chain(m.frame, m.saliency)
    one = m.take(k)
    two = synth.concat_points([one, synth.Points(one.frame.copy(), one.x.copy(), one.y.copy(),
                                                 one.saliency * 0.5, one.feat.copy())])
    p = wl.params()
    _, _, S2, _ = oracle.detect_chains([two], 2, wl.scenes[0], p, 0, 9, 4, 60)
    _, _, S1, _ = oracle.detect_chains([one], 1, wl.scenes[0], p, 0, 9, 4, 60)
    assert np.allclose(S2, S1, rtol=0, atol=1e-12)
