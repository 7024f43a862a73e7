"""GPU-vs-oracle comparison (SURVEY.md §8(c.4) "GPU vs oracle", BASELINE.json north_star):

  * assignments bit-exact;
  * |E_gpu - E_ora| <= 1e-6 + 1e-5 |E_ora|  (same for the appearance distance A);
  * near-tie rule: if z_gpu != z_ora, accept iff z_gpu is feasible and the
    oracle's fp64 energy of z_gpu meets the same bound against E*_ora.
"""
from __future__ import annotations

import numpy as np

import oracle

ATOL, RTOL = 1e-6, 1e-5


def tol(ref):
    return ATOL + RTOL * abs(ref)


class Checker:
    def __init__(self, models_pts, scene_pts, params, first_frame, stride, window):
        self.models = [oracle.model_nodes(m) for m in models_pts]
        self.order, self.scene = oracle.scene_nodes(scene_pts)
        ids = scene_pts.ids()
        self.id2pos = {int(ids[self.order[k]]): k for k in range(self.order.size)}
        self.params = params
        self.first_frame, self.stride, self.window = first_frame, stride, window
        self.scene_pts, self.models_pts = scene_pts, models_pts

    def window_of(self, k):
        o = self.first_frame + k * self.stride
        return oracle.window_range(self.scene.t, o, self.window)

    def oracle_pairs(self, pairs, n_threads=None):
        """Oracle E/A/z for (m, k) pairs; z as caller ids."""
        jm = np.array([m for m, _ in pairs], np.int32)
        wins = [self.window_of(k) for _, k in pairs]
        jb = np.array([w[0] for w in wins], np.int32)
        je = np.array([w[1] for w in wins], np.int32)
        E, Er, A, z = oracle.match_batch(self.models, self.scene, self.params, jm, jb, je, n_threads)
        ids = self.scene_pts.ids()[self.order]
        zid = np.where(z >= 0, ids[np.maximum(z, 0)], -1)
        return E, Er, A, zid

    def check_pair(self, m, k, E_gpu, A_gpu, z_gpu, E_ora, A_ora, z_ora):
        """Returns None if OK, else a message."""
        M = self.models[m].n
        z_gpu = np.asarray(z_gpu[:M], np.int64)
        z_ora = np.asarray(z_ora[:M], np.int64)
        if abs(float(E_gpu) - E_ora) > tol(E_ora):
            return f"E mismatch (m={m},k={k}): gpu {E_gpu} oracle {E_ora}"
        if np.array_equal(z_gpu, z_ora):
            if abs(float(A_gpu) - A_ora) > tol(A_ora):
                return f"A mismatch (m={m},k={k}): gpu {A_gpu} oracle {A_ora}"
            return None
        # near-tie rule
        wb, we = self.window_of(k)
        win = self.scene.slice(wb, we)
        zl = np.array([-1 if v < 0 else self.id2pos[int(v)] - wb for v in z_gpu], np.int32)
        if np.any((zl < -1) | (zl >= we - wb)):
            return f"z outside window (m={m},k={k}): {z_gpu}"
        if not oracle.feasible(self.models[m], win, self.params, zl):
            return f"infeasible gpu assignment (m={m},k={k}): {z_gpu}"
        Ez = oracle.energy(self.models[m], win, self.params, zl)
        if abs(Ez - E_ora) > tol(E_ora):
            return f"assignment differs beyond a near-tie (m={m},k={k}): E(z_gpu)={Ez} E*={E_ora}"
        return "TIE"
