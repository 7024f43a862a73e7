"""C4 (M=200, W=400, stride 10) at large T: batched K-DP vs the v0 reference kernels."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1505_00581_b200 import hgm  # noqa: E402

nf = int(sys.argv[1]) if len(sys.argv) > 1 else 600
for T in [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "10,20,40,80").split(",")]:
    wl = synth.make_workload("C4", T=T, n_frames=nf)
    p = wl.params()
    s = hgm.build_scene_index(wl.scenes[0], device=0, T_max=T)
    models = [hgm.build_model_graph(m, device=0) for m in wl.models]
    res = {}
    for kern in ("v1", "v0"):
        os.environ["HGM_KERNEL"] = kern
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        try:
            res[kern] = hgm.detect_actions(models, s, p, wl.first[0], wl.stride, wl.count[0], wl.window,
                                           want_E_all=True)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            print(f"T={T} {kern}: {dt * 1000:.1f} ms", flush=True)
        except Exception as e:  # noqa: BLE001
            print(f"T={T} {kern}: FAILED {e}", flush=True)
    if "v0" in res and "v1" in res:
        a, b = res["v0"].E_all, res["v1"].E_all
        print(f"T={T}: pairs {a.numel()}, bit-identical E: {bool(torch.equal(a, b))}, "
              f"winners equal: {bool(torch.equal(res['v0'].winner, res['v1'].winner))}", flush=True)
