"""Oracle pins for the single-large-instance regime (PAPER.md
L668-676 Table 3, L752-753 'No restrictions (T = +inf)'): one model against a
whole scene video in one window, T up to unpruned."""
import numpy as np
import pytest

import oracle
import synth
from tests._tiny import tiny_instance


@pytest.mark.parametrize("seed", range(40))
def test_unpruned_T_equals_brute_force(seed):
    """T larger than the scene's frame span removes the closeness constraint (Eq. 8):
    the DP optimum equals the DFS brute force over the causality-only feasible set."""
    model, scene, p = tiny_instance(1000 + seed, M_range=(1, 5), S_range=(1, 8), frames=12)
    p["T"] = int(scene.t.max() - scene.t.min()) + 2 if scene.n else 2
    E, Er, A, z = oracle.match(model, scene, p)
    Eb, zb, _ = oracle.brute(model, scene, p, prune=True)
    assert abs(E - Eb) <= 1e-12 * max(1.0, abs(Eb))
    assert abs(Er - E) <= 1e-9 * max(1.0, abs(E))


def test_energy_non_increasing_in_T_and_saturates():
    """Relaxing the warp bound T enlarges the feasible set (Eq. 8), so E*(T) is
    non-increasing, and constant once T exceeds the window's frame span."""
    wl = synth.make_single(3, n_frames=50, n_nodes=56, model_frames=8, plant=False)
    p = wl.params()
    Es = []
    for T in (2, 3, 5, 10, 20, 51, 52, 200):
        p["T"] = T
        Es.append(oracle.detect(wl.models, wl.scenes[0], p, 0, 1, 1, wl.window).E[0, 0])
    assert all(b <= a + 1e-12 for a, b in zip(Es, Es[1:])), Es
    assert Es[-1] == Es[-2] == Es[-3]


def test_golden_f2_unpruned_fixture_is_consistent():
    """tests/golden/f2_single1_Tinf.json (tools/make_golden_f2.py, oracle only) holds the
    fp64 optimum of the paper's single large instance at T = +inf: its
    assignment is feasible, its energy recomputed from scratch by oracle.energy (Eq. 1,
    not the DP) equals the stored E*, and A = sum of Eq. 2 over the labels (R14)."""
    import json
    import os

    import numpy as np

    import oracle
    import synth

    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "f2_single1_Tinf.json")))
    wl = synth.make_single(1, plant=False)
    model = oracle.model_nodes(wl.models[0])
    order, scene = oracle.scene_nodes(wl.scenes[0])
    wb, we = oracle.window_range(scene.t, 0, wl.window)
    win = scene.slice(wb, we)
    ids = wl.scenes[0].ids()[order]
    pos = {int(ids[k]): k for k in range(ids.size)}
    z = np.array([-1 if v < 0 else pos[v] - wb for v in gold["z_ids"]], np.int32)
    p = dict(gold["params"])
    assert gold["M"] == model.n and gold["S"] == we - wb
    assert oracle.feasible(model, win, p, z)
    assert abs(oracle.energy(model, win, p, z) - gold["E"]) <= 1e-9 * max(1.0, gold["E"])
    A = sum(p["w_dummy"] if z[i] < 0 else float(np.linalg.norm(model.f[i] - win.f[z[i]])) for i in range(model.n))
    assert abs(A - gold["A"]) <= 1e-9 * max(1.0, gold["A"])
    # the unpruned optimum cannot exceed the T = 80 optimum (E* non-increasing in T)
    E80 = oracle.match(model, win, dict(p, T=80))[0]
    assert gold["E"] <= E80 + 1e-9
