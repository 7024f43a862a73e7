"""Writes tests/golden/f2_single1_Tinf.json: the fp64 oracle's result for the paper's
single large instance at T = +inf (Table 3's 1853 ms row; L752-753):
ONE M=30 model vs a whole 754-node / 723-frame scene (synth.make_single(1, plant=False)),
one window covering the video, T = 724 (> the frame span, i.e. unpruned).  Calls only
oracle/ (and the seeded input generator); ~5 minutes on one core.  The GPU test
test_single_instance_unpruned_full_size compares libhgm.so against this file."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import synth  # noqa: E402

wl = synth.make_single(1, plant=False)
p = wl.params()
p["T"] = 724
model = oracle.model_nodes(wl.models[0])
order, scene = oracle.scene_nodes(wl.scenes[0])
wb, we = oracle.window_range(scene.t, 0, wl.window)
t0 = time.time()
E, Er, A, z = oracle.match(model, scene.slice(wb, we), p)
ids = wl.scenes[0].ids()[order]
zid = [int(ids[wb + v]) if v >= 0 else -1 for v in z]
out = dict(source="tools/make_golden_f2.py (oracle.match, fp64), synth.make_single(1, plant=False), T=724, "
                  "window = whole 723-frame video", params=p, M=int(model.n), S=int(we - wb), E=E, E_recomputed=Er,
           A=A, z_ids=zid, oracle_seconds=time.time() - t0)
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                    "f2_single1_Tinf.json")
with open(path, "w") as fh:
    json.dump(out, fh, indent=1)
print(path, E, A, out["oracle_seconds"])
