"""f4 measurement: streaming detection latency (60-frame blocks,
~3 ms per frame for 50 models without overlap, 6 ms with overlapping blocks, vs the
40 ms real-time limit at 25 fps).  A C3-shaped scene is pushed `hop` frames at a time
through hgm.Stream (host points in, host results out: H2D, scene index, unary table,
K-DP, K-BT, argmin and the D2H read are all inside each push); the wall time of every
push is recorded after a warm-up.  One JSON line per (models, hop, stride)."""
import argparse
import json
import time

import numpy as np

import synth
from paper_1505_00581_b200 import hgm as H

ap = argparse.ArgumentParser()
ap.add_argument("--frames", type=int, default=3000)
ap.add_argument("--warmup-frames", type=int, default=300)
a = ap.parse_args()
wl = synth.make_workload("C3", n_frames=a.frames + a.warmup_frames + 60)
sc = wl.scenes[0]
p = wl.params()
protos = [synth.gen_model(c, 30, 2, synth.F_KTH, "stream-protos", s) for c in range(6) for s in range(8)]
dicts = {6: wl.models, 48: protos}
order = np.argsort(sc.frame, kind="stable")
fr_sorted = sc.frame[order]
for n_models, hop, stride in [(6, 1, 1), (6, 30, 1), (6, 60, 60), (48, 1, 1), (48, 30, 1), (48, 60, 60)]:
    models = [H.build_model_graph(m, device=0) for m in dicts[n_models]]
    st = H.Stream(models, p, window=60, stride=stride)
    lat, n_off, pushed = [], 0, 0
    total = a.warmup_frames + a.frames
    for f0 in range(0, total, hop):
        lo, hi = np.searchsorted(fr_sorted, [f0, f0 + hop])
        pts = sc.take(np.sort(order[lo:hi]))
        t = time.perf_counter()
        first, w, s = st.push(pts, hop)
        dt = time.perf_counter() - t
        if f0 >= a.warmup_frames:
            lat.append(dt * 1e3)
            n_off += len(w)
            pushed += hop
    lat = np.array(lat)
    print(json.dumps(dict(metric="stream_ms_per_frame", value=round(float(lat.sum() / pushed), 4), unit="ms/frame",
                          higher_is_better=False, n_models=n_models, hop_frames=hop, stride=stride, window=60,
                          pushes=len(lat), frames=pushed, offsets_reported=n_off,
                          push_ms_median=round(float(np.median(lat)), 4),
                          push_ms_p99=round(float(np.percentile(lat, 99)), 4),
                          push_ms_max=round(float(lat.max()), 4),
                          paper_gtx_ms_per_frame="3 (60-frame blocks, 50 models) / 6 (overlapping)",
                          timing="host wall clock around each synchronous push (H2D + all kernels + D2H)")),
          flush=True)
