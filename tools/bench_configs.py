"""§8(d) configuration sweep: pairs/s, K-DP Gcand/s and its
fraction of the 10.5-issue-slot roofline for C1, C2, C4 (T in {10,20,40,80}; rho in
{2,4,8} at T=20) and the paper-equivalent context rows (50 models M=30 vs a 723-frame,
754-node scene: W = stride = 60 and W = 723).  Inputs HBM-resident (scene index and
model graphs built untimed), CUDA events around `steps` detect_actions calls after
`warmup`; SM clock sampled through NVML right after the timed region.  C3 is
bench.py's headline.  One JSON line per row.  `frac` uses the K-DP event time; with two
lanes (C4) those intervals overlap the other lane's work, so read `frac_wall` there
(candidates / whole call time / roofline: a lower bound on the kernel's fraction)."""
import argparse
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_1505_00581_b200 import hgm as H  # noqa: E402
from paper_1505_00581_b200.work import count_work  # noqa: E402

ISSUE_SLOTS_PER_CAND = 10.5
ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=5)
ap.add_argument("--warmup", type=int, default=3)
ap.add_argument("--only", default="")
ap.add_argument("--dp", default="", help="force the K-DP path: fused | window (default: the library's choice)")
a = ap.parse_args()
if a.dp:
    import os

    os.environ["HGM_DP"] = a.dp


def sm_clock():
    try:
        import pynvml

        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(0)
        return float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
    except Exception:
        return 1965.0


def rows():
    wl = synth.make_workload("C1")
    yield "C1", wl.models, [wl.scenes[0]], 1, wl.count[0], 60, wl.params()
    wl = synth.make_workload("C2")
    yield "C2 (25 clips)", wl.models, wl.scenes, 1, wl.count[0], 60, wl.params()
    for T in (10, 20, 40, 80):
        wl = synth.make_workload("C4", T=T)
        yield f"C4 T={T} rho=4", wl.models, [wl.scenes[0]], 10, wl.count[0], 400, wl.params()
    for rho in (2.0, 8.0):
        wl = synth.make_workload("C4", T=20, rho=rho)
        yield f"C4 T=20 rho={rho:g}", wl.models, [wl.scenes[0]], 10, wl.count[0], 400, wl.params()
    ctx = synth.make_single(1, plant=False)
    protos = [synth.gen_model(c, 30, 1, synth.F_KTH, "ctx-protos", s) for c in range(5) for s in range(10)]
    p = ctx.params()
    yield "context: 50 models x 754-node scene, W=stride=60", protos, ctx.scenes, 60, 12, 60, p
    yield "context: 50 models x 754-node scene, W=723", protos, ctx.scenes, 1, 1, 723, p
    sg = synth.make_single(0, plant=True)
    yield "f2 single instance 754 nodes, T=10", sg.models, sg.scenes, 1, 1, 723, sg.params()
    yield "f2 single instance 754 nodes, T=inf", sg.models, sg.scenes, 1, 1, 723, dict(sg.params(), T=724)


for name, models_pts, scenes_pts, stride, count, W, p in rows():
    if a.only and a.only not in name:
        continue
    models = [H.build_model_graph(m, device=0) for m in models_pts]
    scenes = [H.build_scene_index(s, device=0, T_max=p["T"]) for s in scenes_pts]
    Ms = [len(np.unique(m.frame)) for m in models_pts]

    def run():
        for sc in scenes:
            H.detect_actions(models, sc, p, 0, stride, count, W)

    for _ in range(a.warmup):
        run()
    H.set_profiling(True)
    H.get_stats(reset=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.steps):
        run()
    e1.record()
    torch.cuda.synchronize()
    f = sm_clock()
    st = H.get_stats(reset=True)
    H.set_profiling(False)
    ms = e0.elapsed_time(e1) / a.steps
    cand = 0
    for s in scenes_pts:
        wk = count_work(s.frame, 0, stride, count, W, p["T"])
        cand += wk.real_candidates * sum(max(M - 2, 0) for M in Ms)
    dp_ms = st["ms"]["dp"] / a.steps
    pairs = len(models) * count * len(scenes)
    roof = 148 * 128 * f * 1e6 / ISSUE_SLOTS_PER_CAND / 1e9
    ach = cand / (dp_ms / 1e3) / 1e9 if dp_ms > 0 else 0.0
    print(json.dumps(dict(config=name, dp_path=a.dp or "auto", pairs=pairs, ms_per_call=round(ms, 4), pairs_per_s=round(pairs / ms * 1e3, 1),
                          dp_ms=round(dp_ms, 4), dp_share=round(dp_ms / ms, 3), real_candidates=int(cand),
                          dp_gcand_s=round(ach, 1), roofline_gcand_s=round(roof, 1), frac=round(ach / roof, 4),
                          frac_wall=round(cand / (ms / 1e3) / 1e9 / roof, 4),
                          sm_mhz=f, kernel_ms={k: round(v / a.steps, 4) for k, v in st["ms"].items() if v},
                          l2="no flush between calls (configs re-read their inputs; C2/C4 exceed L2 only partly)")),
          flush=True)
    del models, scenes
