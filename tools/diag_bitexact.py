"""Diagnostic: where do the batched K-DP energies differ from the v0 reference kernels?"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1505_00581_b200 import hgm  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
wl = synth.make_workload(name)
p = wl.params()
s = hgm.build_scene_index(wl.scenes[0], device=0, T_max=p["T"])
models = [hgm.build_model_graph(m, device=0) for m in wl.models]
res = {}
for kern in ("v0", "v1"):
    os.environ["HGM_KERNEL"] = kern
    res[kern] = hgm.detect_actions(models, s, p, wl.first[0], wl.stride, wl.count[0], wl.window, want_E_all=True)
    torch.cuda.synchronize()
a, b = res["v0"].E_all, res["v1"].E_all
bad = (a != b).nonzero()
print("mismatches", bad.shape[0], "of", a.numel())
for m, o in bad[:20].tolist():
    print(f"model {m} offset {o}: v0 {a[m, o].item():.7f} v1 {b[m, o].item():.7f}")
