import os, sys, time
sys.path.insert(0, '/root/repo')
import torch, numpy as np
import bench
from paper_1505_00581_b200 import hgm
wl = bench.rank_workload("C3", 0, 1, 25000)
p = wl["params"]; dev = torch.device("cuda", 0)
scene_d = hgm.DevicePoints.from_host(wl["scene"], device=dev)
models_d = [hgm.DevicePoints.from_host(m, device=dev) for m in wl["models"]]
count = wl["count"]
winner = torch.empty(count, dtype=torch.int32, device=dev); score = torch.empty(count, dtype=torch.float32, device=dev)
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
for it in range(14):
    t = [time.perf_counter()]
    flush.zero_()
    scene = hgm.build_scene_index(scene_d, T_max=p["T"]); t.append(time.perf_counter())
    models = [hgm.build_model_graph(m) for m in models_d]; t.append(time.perf_counter())
    hgm.detect_actions(models, scene, p, wl["first"], 1, count, 60, out=(winner, score, None)); t.append(time.perf_counter())
    del scene, models; t.append(time.perf_counter())
    torch.cuda.synchronize(); t.append(time.perf_counter())
    print(it, " ".join(f"{1000*(t[j+1]-t[j]):8.1f}" for j in range(len(t)-1)), f"total {1000*(t[-1]-t[0]):8.1f}", flush=True)
