"""Seeded tiny random instances for the oracle pins (inputs only, no method arithmetic)."""
import numpy as np

from oracle import NodeSet


def tiny_instance(seed, M_range=(1, 5), S_range=(1, 7), F_range=(1, 3), T_range=(1, 5),
                  wd_choices=(0.1, 0.5, 1.0, 3.0), frames=None, px=8):
    rng = np.random.default_rng(seed)
    M = int(rng.integers(M_range[0], M_range[1] + 1))
    S = int(rng.integers(S_range[0], S_range[1] + 1))
    F = int(rng.integers(F_range[0], F_range[1] + 1))
    T = int(rng.integers(T_range[0], T_range[1] + 1))
    wd = float(rng.choice(wd_choices))
    nfr = frames if frames is not None else max(2, S)
    mt = np.sort(rng.choice(np.arange(0, 2 * M + 2), size=M, replace=False)).astype(np.int32)
    st = np.sort(rng.integers(0, nfr, size=S)).astype(np.int32)
    model = NodeSet(mt, rng.integers(0, px, M).astype(float), rng.integers(0, px, M).astype(float),
                    rng.random((M, F)))
    scene = NodeSet(st, rng.integers(0, px, S).astype(float), rng.integers(0, px, S).astype(float),
                    rng.random((S, F)))
    params = dict(lambda1=float(rng.choice([0.6, 1.0])), lambda2=float(rng.choice([0.2, 0.5])),
                  lambda3=float(rng.choice([5.0, 1.0])), w_dummy=wd, T=T)
    return model, scene, params


def as_dict(ns: NodeSet):
    return dict(t=[int(v) for v in ns.t], x=[float(v) for v in ns.x], y=[float(v) for v in ns.y],
                f=[list(map(float, r)) for r in ns.f])
