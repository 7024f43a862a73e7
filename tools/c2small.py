import os, sys
sys.path.insert(0, '/root/repo')
import torch, synth
from paper_1505_00581_b200 import hgm
wl = synth.make_workload("C2")
p = wl.params()
s = hgm.build_scene_index(wl.scenes[0], device=0, T_max=10)
models = [hgm.build_model_graph(m, device=0) for m in wl.models]
r = hgm.detect_actions(models, s, p, 0, 1, 60, wl.window, want_E_all=True)
torch.cuda.synchronize()
print("ok", r.E_all[:, :4])
