"""Diagnostic: wall-clock breakdown of one bench step (device inputs vs host inputs)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1505_00581_b200 import hgm  # noqa: E402


def main():
    frames = int(sys.argv[1]) if len(sys.argv) > 1 else 25000
    wl = bench.rank_workload("C3", 0, 1, frames)
    p = wl["params"]
    dev = torch.device("cuda", 0)
    scene_d = hgm.DevicePoints.from_host(wl["scene"], device=dev)
    models_d = [hgm.DevicePoints.from_host(m, device=dev) for m in wl["models"]]
    count = wl["count"]
    winner = torch.empty(count, dtype=torch.int32, device=dev)
    score = torch.empty(count, dtype=torch.float32, device=dev)

    def timed(name, fn):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = fn()
        torch.cuda.synchronize()
        print(f"  {name:28s} {1000 * (time.perf_counter() - t0):9.2f} ms", flush=True)
        return r

    for it in range(3):
        print(f"device-input step {it}")
        scene = timed("build_scene_index(dev)", lambda: hgm.build_scene_index(scene_d, T_max=p["T"]))
        models = timed("build_model_graph(dev) x6", lambda: [hgm.build_model_graph(m) for m in models_d])
        timed("detect_actions", lambda: hgm.detect_actions(models, scene, p, wl["first"], 1, count, 60,
                                                          out=(winner, score, None)))
        timed("free handles", lambda: (models.clear(), scene.__del__()))
    for it in range(2):
        print(f"host-input step {it}")
        scene = timed("build_scene_index(host)", lambda: hgm.build_scene_index(wl["scene"], 0, T_max=p["T"]))
        models = timed("build_model_graph(host) x6", lambda: [hgm.build_model_graph(m, 0) for m in wl["models"]])
        timed("detect_actions", lambda: hgm.detect_actions(models, scene, p, wl["first"], 1, count, 60,
                                                          device_out=False))


if __name__ == "__main__":
    main()
