"""Algorithmic work of the recursion, counted on the host from the frame
histogram (the roofline numerator of bench.py).

Per (model, offset) instance and per recursion step i = 3..M (Eq. 10):
  * real states (b, a): pairs with t'(a) < t'(b) < t'(a) + T inside the window
    (the admissible cross-section of);
  * real-triple candidates: for each real state, the nodes c with
    t'(b) < t'(c) < t'(a) + T inside the window (R1/R2);
  * dummy-form states (b, eps), (eps, a), (eps, eps) and their candidates.
One real-triple candidate is the unit of the ALU roofline ("min-plus op").
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class Work:
    real_candidates: int  # per step, summed over offsets
    real_states: int
    eps_states: int
    eps_candidates: int
    windows: int

    def times(self, k: int) -> "Work":
        return Work(self.real_candidates * k, self.real_states * k, self.eps_states * k, self.eps_candidates * k,
                    self.windows)


def count_work(frames, first_frame: int, stride: int, count: int, window: int, T: int,
               per_offset: bool = False):
    """Exact counts for one model step over `count` offsets of a scene whose
    (unsorted or sorted) integer frames are `frames`.  per_offset=True returns the
    real-triple candidates of every offset (int64 [count]) instead of the totals."""
    frames = np.asarray(frames, dtype=np.int64)
    if count <= 0 or frames.size == 0:
        return np.zeros(max(count, 0), np.int64) if per_offset else Work(0, 0, 0, 0, max(count, 0))
    offs = first_frame + stride * np.arange(count, dtype=np.int64)
    lo_f = int(min(offs.min(), frames.min())) - T - 1
    hi_f = int(max(offs.max() + window, frames.max())) + T + 2
    hist = np.bincount(frames - lo_f, minlength=hi_f - lo_f + 1).astype(np.int64)
    cum = np.concatenate([[0], np.cumsum(hist)])  # cum[f - lo_f] = #nodes with frame < f

    def n_at(f):  # nodes in frame f (vector)
        return hist[f - lo_f]

    def below(f):  # nodes with frame < f
        return cum[np.clip(f - lo_f, 0, cum.size - 1)]

    rc = np.zeros(count, np.int64)
    rs = np.zeros(count, np.int64)
    ec = np.zeros(count, np.int64)
    wend = offs + window
    for rb in range(window):
        fb = offs + rb
        nb = n_at(fb)
        # (b, eps) candidates: frames (fb, min(fb+T, wend))
        ec += nb * (below(np.minimum(fb + T, wend)) - below(fb + 1))
        # (eps, a) candidates with a = b-frame: identical count
        ec += nb * (below(np.minimum(fb + T, wend)) - below(fb + 1))
        for j in range(1, min(T, rb + 1)):
            fa = fb - j
            na = n_at(fa)
            st = nb * na
            rs += st
            rc += st * np.maximum(below(np.minimum(fa + T, wend)) - below(fb + 1), 0)
    if per_offset:
        return rc
    sw = below(wend) - below(offs)
    es = 2 * sw + 1
    ec += sw  # (eps, eps) scans the whole window
    return Work(int(rc.sum()), int(rs.sum()), int(es.sum()), int(ec.sum()), count)
