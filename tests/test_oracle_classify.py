"""Oracle pins for the recognition layer: nearest prototype
classifier on the appearance distance (§4) per scene block
(L739-743) and the majority vote over blocks (SPEC, D-12 / vote reading R-f1b)."""
import numpy as np
import pytest

import oracle
import synth


@pytest.mark.parametrize("labels,expect", [
    ([], -1), ([-1, -1], -1), ([3], 3), ([0, 1, 1, 2, 1], 1), ([2, 2, 0, 0], 0), ([5, -1, 5, 4, 4, -1], 4),
    ([1, 0, 2, 2, 1, 0], 0), ([7, 7, 7, -1, -1, -1, -1], 7)])
def test_majority_vote_hand_cases(labels, expect):
    assert oracle.majority_vote(labels) == expect


def test_majority_vote_brute_force():
    """Against the definition: the label with the most votes, the smallest among ties."""
    rng = np.random.default_rng(0)
    for _ in range(300):
        v = rng.integers(-1, 4, size=int(rng.integers(0, 12)))
        cand = [l for l in range(4) if (v == l).sum() > 0]
        want = -1 if not cand else sorted(cand, key=lambda l: (-(v == l).sum(), l))[0]
        assert oracle.majority_vote(v) == want


def _small(seed, **kw):
    return synth.make_recognition(seed, n_classes=3, protos_per_class=1, count=4, block=20, model_frames=8,
                                  pts_per_frame=1, F=8, rho=1.0, T=5, **kw)


def _classify(rs, protos=None, labels=None, threshold=float("inf")):
    protos = rs.prototypes if protos is None else protos
    labels = rs.labels if labels is None else labels
    return oracle.classify_blocks(protos, labels, rs.scene, rs.params(), 0, rs.stride, rs.count, rs.block,
                                  threshold=threshold)


@pytest.mark.parametrize("seed", range(3))
def test_exact_copy_is_recognised_with_distance_zero(seed):
    """A block holding an exact copy of a prototype has appearance distance 0 to it
    (E* = 0 is the global minimum of a sum of non-negative terms, so A = 0) and,
    no other prototype being at distance 0, takes that prototype's label."""
    rs = _small(seed, exact=True)
    r = _classify(rs)
    for k in range(rs.count):
        c = int(rs.truth[k])
        assert r.A[c, k] == 0.0
        assert (r.A[np.arange(len(rs.prototypes)) != c, k] > 0).all()
    assert np.array_equal(r.block_label, rs.truth)
    assert np.all(r.block_score == 0.0)
    assert r.clip_label == oracle.majority_vote(rs.truth)


def test_single_prototype_dictionary_takes_its_label():
    rs = _small(1)
    r = _classify(rs, protos=rs.prototypes[1:2], labels=[7])
    assert np.all(r.block_label == 7) and r.clip_label == 7
    assert np.array_equal(r.block_score, r.A[0])


def test_duplicate_prototype_tie_goes_to_lowest_index():
    """Identical prototypes have identical distances; D-12 picks the lower index."""
    rs = _small(2)
    p = rs.prototypes
    r = _classify(rs, protos=[p[0], p[0], p[1]], labels=[4, 2, 1])
    a = r.A
    assert np.array_equal(a[0], a[1])
    for k in range(rs.count):
        want = 4 if a[0, k] <= a[2, k] else 1
        assert r.block_label[k] == want


def test_appending_a_farther_prototype_keeps_labels():
    """SPEC invariant: a prototype whose distance is strictly larger than the current
    nearest one cannot change a block's label."""
    rs = _small(3)
    base = _classify(rs, protos=rs.prototypes[:2], labels=rs.labels[:2])
    full = _classify(rs)
    far = full.A[2] > base.block_score
    assert far.any()
    assert np.array_equal(full.block_label[far], base.block_label[far])


def test_threshold_abstains_and_vote_ignores_unlabelled():
    rs = _small(4, exact=True, class_of_block=lambda k: [0, 0, 1, 2][k])
    r_all = _classify(rs)
    assert r_all.clip_label == 0
    thr = float(np.sort(r_all.block_score)[-1]) / 2 if r_all.block_score.max() > 0 else 0.0
    r = _classify(rs, threshold=thr)
    assert np.array_equal(r.block_label, np.where(r_all.block_score <= thr, r_all.block_label, -1))
    assert r.clip_label == oracle.majority_vote(r.block_label)
