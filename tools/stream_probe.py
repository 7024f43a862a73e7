"""Where a frame-by-frame stream push spends its time: scene index build vs the detect
call (48 models, one offset), host wall clock, median of 200."""
import time

import numpy as np
import torch

import synth
from paper_1505_00581_b200 import hgm as H

wl = synth.make_workload("C3", n_frames=400)
sc = wl.scenes[0]
p = wl.params()
protos = [synth.gen_model(c, 30, 2, synth.F_KTH, "stream-protos", s) for c in range(6) for s in range(8)]
for nm in (6, 48):
    models = [H.build_model_graph(m, device=0) for m in (wl.models if nm == 6 else protos)]
    tb, td = [], []
    for k in range(200):
        sel = np.nonzero((sc.frame >= k) & (sc.frame < k + 60))[0]
        pts = sc.take(sel)
        pts.frame = pts.frame - k
        t0 = time.perf_counter()
        s = H.build_scene_index(pts, device=0, T_max=10)
        t1 = time.perf_counter()
        H.detect_actions(models, s, p, 0, 1, 1, 60, device_out=False)
        t2 = time.perf_counter()
        tb.append(t1 - t0)
        td.append(t2 - t1)
    H.set_profiling(True)
    H.get_stats(reset=True)
    H.detect_actions(models, s, p, 0, 1, 1, 60, device_out=False)
    st = H.get_stats(reset=True)
    H.set_profiling(False)
    print(nm, "models: scene build ms", round(np.median(tb) * 1e3, 3), "detect ms", round(np.median(td) * 1e3, 3),
          {k: round(v, 3) for k, v in st["ms"].items() if v}, st["launches"])
