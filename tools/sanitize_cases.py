"""Small end-to-end cases for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): C0 seeds, C1 offsets, a C2 clip (6-model batch), small C4 at T = 80 (a-frame
chunks, single-stage items), a single 754-node instance at T = 10, detect with both score
modes.  Each case runs through the C ABI and is compared against the oracle on a few pairs
so a sanitizer-silent but wrong run also fails.  usage: python tools/sanitize_cases.py [case...]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_1505_00581_b200 import hgm as H  # noqa: E402
from tests._parity import Checker  # noqa: E402


def run(wl, scene_idx=0, ks=None, models=None, count=None):
    p = wl.params()
    count = count or wl.count[scene_idx]
    scene = H.build_scene_index(wl.scenes[scene_idx], device=0, T_max=p["T"])
    mids = list(range(len(wl.models))) if models is None else models
    mh = [H.build_model_graph(wl.models[m], device=0) for m in mids]
    det = H.detect_actions(mh, scene, p, wl.first[scene_idx], wl.stride, count, wl.window, want_E_all=True,
                           device_out=False)
    det1 = H.detect_actions(mh, scene, p, wl.first[scene_idx], wl.stride, count, wl.window, score_mode=1,
                            device_out=False)
    r = H.match_model_at_offsets(mh[0], scene, p, wl.first[scene_idx], wl.stride, count, wl.window,
                                 device_out=False)
    chk = Checker([wl.models[m] for m in mids], wl.scenes[scene_idx], p, wl.first[scene_idx], wl.stride, wl.window)
    ks = ks or [0, count // 2, count - 1]
    E_o, _, A_o, z_o = chk.oracle_pairs([(0, k) for k in ks])
    for j, k in enumerate(ks):
        msg = chk.check_pair(0, k, r.E[k], r.A[k], r.z[k], E_o[j], A_o[j], z_o[j])
        assert msg in (None, "TIE"), msg
        assert abs(det.E_all[0, k] - r.E[k]) <= 1e-6 + 1e-5 * abs(r.E[k])
    assert det1.score.shape == det.score.shape
    return count


def _c4_short(T, M, nf):
    wl = synth.make_workload("C4", T=T, n_frames=nf)
    wl.models = [m.take(np.nonzero(m.frame <= np.unique(m.frame)[M - 1])[0]) for m in wl.models]
    return wl


def _many_models():
    wl = synth.make_workload("C2")
    wl.models = wl.models * 3  # 18 models of equal M: batches of 8, 8, 2 on three lanes
    return wl


CASES = {
    "c0": lambda: [run(synth.make_workload("C0", seed=s)) for s in range(3)],
    "c1": lambda: run(synth.make_workload("C1"), count=120, ks=[0, 60, 119]),
    "c2": lambda: run(synth.make_workload("C2"), scene_idx=3, count=60, ks=[0, 30, 59]),
    "c4t80": lambda: run(_c4_short(80, 10, 420), models=[0, 1], ks=[0]),
    "single": lambda: run(synth.make_single(0, plant=True), ks=[0]),
    "lanes": lambda: run(_many_models(), scene_idx=2, count=40, ks=[0, 39]),  # 3 concurrent model batches
}

if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for n in names:
        CASES[n]()
        print("case", n, "ok", flush=True)
