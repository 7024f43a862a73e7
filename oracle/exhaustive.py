"""Pure-Python exhaustive (S+1)^M enumeration.  TEST INFRASTRUCTURE ONLY.

Written independently of hgm_oracle.c / hgm_brute.c (different language, no
shared helpers) straight from SURVEY.md §8(c.1): the energy of PAPER.md Eq. 1
(L117) with U of Eq. 2 (L126-137), D of Eqs. 3-6 (L139-165), the dummy rule
A5, and the feasible set of Eqs. 7-8 under readings A1/A2.  For M <= 5,
S <= 7 only; it pins the DFS enumerator and the DP.
"""
from __future__ import annotations

import itertools
import math

EPS = None  # the dummy label


def unary(fm, fs, w_dummy):
    """Eq. 2."""
    if fs is None:
        return w_dummy
    return math.sqrt(sum((a - b) ** 2 for a, b in zip(fm, fs)))


def angle(p, v, q):
    """Angle at the middle point v between v->p and v->q, in [0, pi]; 0 on a
    zero-length ray (A8, A10).  Uses acos of the normalised dot product -- a
    different formula from the C oracle's atan2(|cross|, dot)."""
    ux, uy = p[0] - v[0], p[1] - v[1]
    wx, wy = q[0] - v[0], q[1] - v[1]
    nu = math.hypot(ux, uy)
    nw = math.hypot(wx, wy)
    if nu == 0.0 or nw == 0.0:
        return 0.0
    c = (ux * wx + uy * wy) / (nu * nw)
    return math.acos(max(-1.0, min(1.0, c)))


def circ(d):
    """Circular difference, in [-pi, pi]."""
    return math.atan2(math.sin(d), math.cos(d))


def distortion(mt, mp, st, sp, lambda3):
    """D for model triple (i, i-1, i-2) with times mt, points mp and scene
    triple (z_i, z_{i-1}, z_{i-2}) with times st, points sp (Eqs. 3-6)."""
    dt = abs((mt[0] - mt[1]) - (st[0] - st[1])) + abs((mt[1] - mt[2]) - (st[1] - st[2]))
    e1 = circ(angle(mp[0], mp[1], mp[2]) - angle(sp[0], sp[1], sp[2]))
    e2 = circ(angle(mp[1], mp[0], mp[2]) - angle(sp[1], sp[0], sp[2]))
    return dt + lambda3 * math.sqrt(e1 * e1 + e2 * e2)


def energy(model, scene, params, z):
    """Eq. 1 on the chain (L117, L200), lambdas explicit; z entries are scene
    indices or None (dummy)."""
    l1, l2, l3, wd = params["lambda1"], params["lambda2"], params["lambda3"], params["w_dummy"]
    E = 0.0
    M = len(model["t"])
    for i in range(M):
        fs = None if z[i] is EPS else scene["f"][z[i]]
        E += l1 * unary(model["f"][i], fs, wd)
        if i >= 2 and all(z[k] is not EPS for k in (i, i - 1, i - 2)):
            mt = [model["t"][k] for k in (i, i - 1, i - 2)]
            mp = [(model["x"][k], model["y"][k]) for k in (i, i - 1, i - 2)]
            st = [scene["t"][z[k]] for k in (i, i - 1, i - 2)]
            sp = [(scene["x"][z[k]], scene["y"][z[k]]) for k in (i, i - 1, i - 2)]
            E += l2 * distortion(mt, mp, st, sp, l3)
    return E


def feasible(scene, T, z):
    """pair rule on (z1, z2); triple rule for every real z_i,
    i >= 3, against the nearest real labels among z_{i-1}, z_{i-2}."""
    t = scene["t"]
    M = len(z)
    if M >= 2 and z[0] is not EPS and z[1] is not EPS:
        if not (t[z[0]] < t[z[1]] < t[z[0]] + T):
            return False
    for i in range(2, M):
        c, b, a = z[i], z[i - 1], z[i - 2]
        if c is EPS:
            continue
        if b is not EPS and a is not EPS:
            ok = t[b] < t[c] < t[a] + T
        elif b is EPS and a is not EPS:
            ok = t[a] < t[c] < t[a] + T
        elif b is not EPS and a is EPS:
            ok = t[b] < t[c] < t[b] + T
        else:
            ok = True
        if not ok:
            return False
    return True


def exhaustive_match(model, scene, params):
    """min over the feasible set, first minimum in lexicographic order with the
    label order 0 < 1 < ... < S-1 < eps (A11).  Returns (E, z, n_feasible)."""
    S = len(scene["t"])
    labels = list(range(S)) + [EPS]
    best, zbest, nfeas, second = math.inf, None, 0, math.inf
    for z in itertools.product(labels, repeat=len(model["t"])):
        if not feasible(scene, params["T"], z):
            continue
        nfeas += 1
        E = energy(model, scene, params, z)
        if E < best:
            best, zbest, second = E, z, best
        elif E < second:
            second = E
    return best, [(-1 if v is EPS else v) for v in zbest], nfeas, second
