"""Host-enqueue vs device time of small detect calls (context rows, f2 T=10, C1): the time
until hgm_detect_actions returns (host enqueue; outputs stay on the device) against the
time until the stream drains.  usage: python tools/ctx_probe.py [row-substring]
(HGM_HOSTPROF=1 with one row: the steady-state host profile of that row, printed at exit)"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_1505_00581_b200 import hgm as H  # noqa: E402

ctx = synth.make_single(1, plant=False)
protos = [synth.gen_model(c, 30, 1, synth.F_KTH, "ctx-protos", s) for c in range(5) for s in range(10)]
sg = synth.make_single(0, plant=True)
c1 = synth.make_workload("C1")
rows = [("context W=60", protos, ctx.scenes[0], 60, 12, 60, ctx.params()),
        ("context W=723", protos, ctx.scenes[0], 1, 1, 723, ctx.params()),
        ("f2 T=10", sg.models, sg.scenes[0], 1, 1, 723, sg.params()),
        ("C1", c1.models, c1.scenes[0], 1, c1.count[0], 60, c1.params())]
only = sys.argv[1] if len(sys.argv) > 1 else ""
for name, mp, sp, stride, count, W, p in rows:
    if only not in name:
        continue
    models = [H.build_model_graph(m, device=0) for m in mp]
    scene = H.build_scene_index(sp, device=0, T_max=p["T"])
    for _ in range(3):
        H.detect_actions(models, scene, p, 0, stride, count, W)
    torch.cuda.synchronize()
    H.get_stats(reset=True)  # (also restarts the HGM_HOSTPROF accumulators: steady state only)
    enq, tot = [], []
    for _ in range(20):
        t0 = time.perf_counter()
        H.detect_actions(models, scene, p, 0, stride, count, W)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        enq.append(t1 - t0)
        tot.append(t2 - t0)
    print(f"{name:14s} host enqueue {1e3 * np.median(enq):7.3f} ms  enqueue+drain {1e3 * np.median(tot):7.3f} ms", flush=True)
