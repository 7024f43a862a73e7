"""f2 probe: one model (M=30) vs a whole 754-node / 723-frame scene, T in a sweep
(Table 3, Fig. curvet).  Times match_model_at_offsets with CUDA events and
checks E / A / z against the oracle where it finishes quickly."""
import sys
import time

import numpy as np
import torch

import oracle
import synth
from paper_1505_00581_b200 import hgm as H

Ts = [int(t) for t in sys.argv[1:] if not t.startswith("-")] or [10, 20, 40, 80, 160, 724]
for T in Ts:
    wl = synth.make_single(0, T=min(T, 10))
    p = wl.params()
    p["T"] = T
    sc = H.build_scene_index(wl.scenes[0], device=0, T_max=T)
    m = H.build_model_graph(wl.models[0], device=0)
    for _ in range(2):
        r = H.match_model_at_offsets(m, sc, p, 0, 1, 1, wl.window, device_out=True)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    n = 5
    ev[0].record()
    for _ in range(n):
        r = H.match_model_at_offsets(m, sc, p, 0, 1, 1, wl.window, device_out=True)
    ev[1].record()
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1]) / n
    E, A = float(r.E.cpu()[0]), float(r.A.cpu()[0])
    if "--stats" in sys.argv:
        H.set_profiling(True)
        H.get_stats(reset=True)
        r = H.match_model_at_offsets(m, sc, p, 0, 1, 1, wl.window, device_out=True)
        torch.cuda.synchronize()
        st = H.get_stats(reset=True)
        H.set_profiling(False)
        print({k: round(v, 3) for k, v in st["ms"].items() if v}, st["launches"], st["dp_launches"])
    line = f"T={T:4d} S={wl.scenes[0].n} ms={ms:8.3f} E={E:.6f} A={A:.6f}"
    if T <= 80 or "--oracle" in sys.argv:
        t0 = time.time()
        ref = oracle.detect(wl.models, wl.scenes[0], p, 0, 1, 1, wl.window)
        line += f"  oracle E={ref.E[0,0]:.6f} ({time.time()-t0:.1f}s) dE={abs(E-ref.E[0,0]):.2e}"
    print(line, flush=True)
