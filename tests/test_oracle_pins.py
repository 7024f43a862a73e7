"""Pins of the CPU oracle's energy terms against values the paper / mathematics fix.

Every test here checks the oracle against something other than itself: a worked
example with a hand-derived value, a closed form, or an independent formula.
"""
import math

import numpy as np
import pytest

import oracle
from oracle import NodeSet, exhaustive

L = oracle.lib()


def ns(t, xy, f):
    xy = np.asarray(xy, float)
    return NodeSet(np.asarray(t, np.int32), xy[:, 0].copy(), xy[:, 1].copy(), np.asarray(f, float))


# --- Eq. 2 ------------------------------------------------
def test_unary_345_identity_and_dummy():
    # S:L117-119 worked examples: (3,4) vs (0,0) -> 5; identical -> 0; eps -> W^d
    m = ns([0], [[0, 0]], [[3.0, 4.0]])
    s = ns([0, 1], [[0, 0], [1, 1]], [[0.0, 0.0], [3.0, 4.0]])
    mc, sc = m.cstruct(), s.cstruct()
    assert L.or_unary(mc, 0, sc, 0, 2.5) == 5.0
    assert L.or_unary(mc, 0, sc, 1, 2.5) == 0.0
    assert L.or_unary(mc, 0, sc, 2, 2.5) == 2.5  # label S is the dummy


def test_unary_isometry_invariance():
    # a common orthonormal transform of feature space leaves U unchanged
    rng = np.random.default_rng(1)
    F = 6
    Q, _ = np.linalg.qr(rng.standard_normal((F, F)))
    fm, fs = rng.random((1, F)), rng.random((3, F))
    a = [L.or_unary(ns([0], [[0, 0]], fm).cstruct(), 0, ns([0, 1, 2], np.zeros((3, 2)), fs).cstruct(), n, 1.0)
         for n in range(3)]
    b = [L.or_unary(ns([0], [[0, 0]], fm @ Q).cstruct(), 0, ns([0, 1, 2], np.zeros((3, 2)), fs @ Q).cstruct(),
                    n, 1.0) for n in range(3)]
    np.testing.assert_allclose(a, b, rtol=1e-13)


# --- Eq. 5 ----------------------------------------------------
def test_delta_worked_example():
    # t(i)=3, t(j)=5, t'(z_i)=10, t'(z_j)=14 -> |(-2) - (-4)| = 2
    assert L.or_delta(3, 5, 10, 14) == 2.0
    assert L.or_delta(7, 5, 12, 10) == 0.0
    assert L.or_delta(3, 5, 10, 14) == L.or_delta(5, 3, 14, 10)


# --- Eq. 6 angles ----------------------------------------
def test_angles_closed_forms():
    # perpendicular pi/2, parallel 0, opposite pi (vertex = middle point)
    assert L.or_angle(1, 0, 0, 0, 0, 1) == pytest.approx(math.pi / 2, abs=1e-15)
    assert L.or_angle(2, 0, 0, 0, 5, 0) == 0.0
    assert L.or_angle(-1, 0, 0, 0, 1, 0) == pytest.approx(math.pi, abs=1e-15)
    # A10: a zero-length ray gives 0
    assert L.or_angle(0, 0, 0, 0, 1, 1) == 0.0
    assert L.or_angle(3, 3, 1, 1, 1, 1) == 0.0
    # equilateral triangle: pi/3 at every vertex
    h = math.sqrt(3) / 2
    assert L.or_angle(1, 0, 0, 0, 0.5, h) == pytest.approx(math.pi / 3, abs=1e-15)


def test_angles_agree_with_independent_acos_formula():
    rng = np.random.default_rng(2)
    for _ in range(500):
        p, v, q = rng.integers(-5, 6, size=(3, 2)).astype(float)
        a = L.or_angle(*p, *v, *q)
        b = exhaustive.angle(p, v, q)
        assert abs(a - b) < 1e-7  # acos loses precision near 0/pi; atan2 does not


def test_wrap():
    assert L.or_wrap(0.25) == 0.25
    assert L.or_wrap(2 * math.pi - 0.1) == pytest.approx(-0.1, abs=1e-15)
    assert L.or_wrap(-2 * math.pi + 0.2) == pytest.approx(0.2, abs=1e-15)


def _triangle(alpha, beta):
    """j=(0,0), i=(1,0), k chosen so the angle at j is alpha and at i is beta."""
    ta, tb = math.tan(alpha), math.tan(beta)
    kx = tb / (ta + tb)
    return [(1.0, 0.0), (0.0, 0.0), (kx, kx * ta)]  # (i, j, k)


# --- Eqs. 3-6: D^g and D --------------------------------
def test_dg_worked_example_pi_over_4():
    # model angles (pi/2 at j, pi/4 at i), scene (pi/4, pi/4) -> pi/4
    s = ns([10, 11, 12], [[1, 1], [0, 0], [2, 0]], np.zeros((3, 1)))  # sorted: z_k, z_j, z_i
    # model indices are chain order (k, j, i) = (0, 1, 2); scene (z_k, z_j, z_i) = (0, 1, 2)
    m = ns([0, 1, 2], [[0, 1], [0, 0], [1, 0]], np.zeros((3, 1)))  # k=(0,1), j=(0,0), i=(1,0)
    d = L.or_distortion(m.cstruct(), 2, s.cstruct(), 2, 1, 0, 1.0)
    # equal frame gaps (1,1) vs (1,1): D^t = 0, so D = lambda3 * D^g
    assert d == pytest.approx(math.pi / 4, abs=1e-14)


def test_d_worked_example_3_5():
    # Delta sum 3, lambda3 = 5, angle-difference norm 0.1 -> 3.5
    P = _triangle(0.8, 0.6)  # model: angle 0.8 at j (node i-1), 0.6 at i
    Q = _triangle(0.7, 0.6)  # scene: 0.7 at z_j, 0.6 at z_i  -> e1 = 0.1, e2 = 0
    m = ns([0, 1, 2], [P[2], P[1], P[0]], np.zeros((3, 1)))  # chain order k, j, i
    # model gaps (1, 1); scene gaps (3, 2): Delta(i,j) = |1-3| = 2, Delta(j,k) = |1-2| = 1
    s = ns([0, 2, 5], [Q[2], Q[1], Q[0]], np.zeros((3, 1)))
    d = L.or_distortion(m.cstruct(), 2, s.cstruct(), 2, 1, 0, 5.0)
    assert d == pytest.approx(3.5, abs=1e-12)
    # a dummy anywhere in the triple -> 0 (A5)
    assert L.or_distortion(m.cstruct(), 2, s.cstruct(), 3, 1, 0, 5.0) == 0.0
    assert L.or_distortion(m.cstruct(), 2, s.cstruct(), 2, 3, 0, 5.0) == 0.0
    assert L.or_distortion(m.cstruct(), 2, s.cstruct(), 2, 1, 3, 5.0) == 0.0


def test_distortion_matches_independent_python():
    rng = np.random.default_rng(3)
    for _ in range(300):
        mt = np.sort(rng.choice(20, 3, replace=False))
        st = np.sort(rng.choice(30, 3, replace=False))
        mp = rng.integers(0, 10, (3, 2)).astype(float)
        sp = rng.integers(0, 10, (3, 2)).astype(float)
        m = ns(mt, mp, np.zeros((3, 1)))
        s = ns(st, sp, np.zeros((3, 1)))
        a = L.or_distortion(m.cstruct(), 2, s.cstruct(), 2, 1, 0, 5.0)
        b = exhaustive.distortion(mt[::-1], mp[::-1], st[::-1], sp[::-1], 5.0)
        assert abs(a - b) < 1e-6


def test_distortion_invariances_exact_integer():
    # scene translation, 90-degree rotation, x2 scale, time shift leave D unchanged
    rng = np.random.default_rng(4)
    for _ in range(200):
        mt = np.sort(rng.choice(20, 3, replace=False))
        st = np.sort(rng.choice(30, 3, replace=False))
        mp = rng.integers(0, 10, (3, 2)).astype(float)
        sp = rng.integers(0, 10, (3, 2)).astype(float)
        m = ns(mt, mp, np.zeros((3, 1))).cstruct()
        base = L.or_distortion(m, 2, ns(st, sp, np.zeros((3, 1))).cstruct(), 2, 1, 0, 5.0)
        for sp2, st2 in [(sp + [7, -3], st), (sp[:, ::-1] * [-1, 1], st), (sp * 2, st), (sp, st + 11)]:
            v = L.or_distortion(m, 2, ns(st2, sp2, np.zeros((3, 1))).cstruct(), 2, 1, 0, 5.0)
            assert v == pytest.approx(base, abs=1e-12)


# --- Eq. 1 / Eq. 9 -------------------------------------
def test_all_dummy_energy_closed_form():
    # all-eps assignment -> lambda1 * M * W^d exactly
    rng = np.random.default_rng(5)
    for M in (1, 2, 3, 8):
        m = ns(np.arange(M), rng.random((M, 2)), rng.random((M, 4)))
        s = ns(np.arange(5), rng.random((5, 2)), rng.random((5, 4)))
        p = dict(lambda1=0.6, lambda2=0.2, lambda3=5.0, w_dummy=2.5, T=10)
        assert oracle.energy(m, s, p, [-1] * M) == pytest.approx(0.6 * M * 2.5, rel=1e-15)


def test_exact_copy_energy_zero_and_hand_sum():
    rng = np.random.default_rng(6)
    m = ns([0, 1, 3], rng.integers(0, 50, (3, 2)), rng.random((3, 5)))
    # scene = model shifted by 10 frames: Delta terms vanish
    s = ns([10, 11, 13], np.array([m.x, m.y]).T, m.f)
    p = dict(lambda1=0.6, lambda2=0.2, lambda3=5.0, w_dummy=1.0, T=10)
    assert oracle.energy(m, s, p, [0, 1, 2]) == 0.0
    # hand sum for M=3: lambda1 * (U1 + U2 + U3) + lambda2 * D
    z = [1, -1, 2]
    E = oracle.energy(m, s, p, z)
    hand = 0.6 * (np.linalg.norm(m.f[0] - s.f[1]) + 1.0 + np.linalg.norm(m.f[2] - s.f[2]))
    assert E == pytest.approx(hand, rel=1e-14)


# --- §3.4 minnode and model graph (L198) ----------------
def test_minnode_figure_example():
    # Fig. 6 caption: "frame 8 has nodes 9, 10 and 11" (1-based)
    frames = [1, 2, 3, 4, 5, 6, 7, 7, 8, 8, 8, 10]  # nodes 1..12; frame 8 -> nodes 9..11
    s = ns(frames, np.zeros((12, 2)), np.zeros((12, 1))).cstruct()
    assert L.or_minnode_at(s, 10, 8) + 1 == 9
    assert L.or_minnode_at(s, 10, 9) + 1 == 12  # empty frame 9 -> first node of frame 10 (A4)
    assert L.or_minnode_at(s, 10, 11) == 12  # past the end -> sentinel S
    assert L.or_minnode_at(s, 10, 0) == 0


def test_model_chain_rules():
    # most salient point per frame; empty frames absent (L200)
    idx = oracle.model_chain([5, 5], [0.9, 0.4])
    assert list(idx) == [0]
    idx = oracle.model_chain([4, 1, 2, 1], [0.1, 0.2, 0.3, 0.2])
    assert list(idx) == [1, 2, 0]  # frames (1, 2, 4); tie on frame 1 keeps the earliest
    assert list(oracle.model_chain([7], [0.0])) == [0]  # M = 1


def test_scene_sort_is_stable():
    order = oracle.scene_sorted([3, 1, 3, 1, 2])
    assert list(order) == [1, 3, 4, 0, 2]
