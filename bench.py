#!/usr/bin/env python
"""Benchmark: detect_actions over a KTH-shaped synthetic scene (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl hgm|reference] [--workload C3|C1]

One "step" = one pass of the whole hot path over the
rank's batch: scene index + direction band (a2), model chains (a1), unary
table (a3), state enumeration + recursion (a4-a5), init search + backtrack +
appearance distance (a6), per-offset model argmin (a7), and for N > 1 the
NCCL all_gather of packed per-offset winners.

Workload (weak scaling): every rank owns a C3-shaped slice of one long scene
-- 25,000 frames per GPU at rho = 4 points/frame (~100k points), one planted
action per 200 frames, 6 models of M = 30, W = 60, stride 1, T = 10.  The
scene of N GPUs is N x 25,000 frames; rank r matches offsets
[r*25000, (r+1)*25000) (its windows reach W-1 frames into the next slice).

`value`  : pairs/s with the inputs resident in HBM (device point arrays).
`e2e`    : same through the public host API (pinned host inputs copied in,
           winners and scores copied back, every step).
The oracle (test infrastructure) is executed only for `cpu_baseline` (rank 0,
N = 1) and for `--impl reference`.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BASELINE_METRIC = "matched (model, offset) pairs/sec and frames/sec at 1/2/4/8 B200; % ALU roofline"
ISSUE_SLOTS_PER_CAND = 10.5  # 6 FADD + FMUL + FFMA + MUFU + FFMA + 1/2 FMNMX3
LANES_PER_CLK = 148 * 4 * 32  # 148 SMs x 4 SMSPs x 32 lanes
# XU (MUFU) pipe: 0.497 warp-instructions / clk / SM measured for MUFU.SQRT on this pool's
# B200 (tools/pipe_microbench.cu, profiles/r01_pipe_microbench.txt) = 15.9 lanes / clk / SM;
# every model-candidate needs one square root (Eq. 6's norm), so this is a second, tighter bound.
XU_LANES_PER_CLK = 148 * 0.497 * 32


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="hgm", choices=["hgm", "reference"])
    ap.add_argument("--workload", default="C3", choices=["C3", "C1"])
    ap.add_argument("--frames-per-gpu", type=int, default=25000)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    return ap.parse_args()


# --------------------------------------------------------------------- workload
def rank_workload(name, rank, world, frames_per_gpu):
    import synth

    if name == "C1":  # single GPU only: one model vs one 600-frame clip, all offsets
        wl = synth.make_workload("C1")
        return dict(models=wl.models, scene=wl.scenes[0], first=0, count=wl.count[0], window=wl.window,
                    stride=wl.stride, params=wl.params(), frames=600, desc=dict(
                        workload="C1: 1 model (M=30) x 600-frame clip, rho=2.5, W=60, stride 1, T=10"))
    total = frames_per_gpu * world
    W = 60
    lo = rank * frames_per_gpu
    hi = min(lo + frames_per_gpu + W - 1, total)
    wl = synth.make_workload("C3", n_frames=total, frame_range=(lo, hi))
    n_off_total = total - W + 1
    k_end = min(lo + frames_per_gpu, n_off_total)
    return dict(models=wl.models, scene=wl.scenes[0], first=lo, count=k_end - lo, window=W, stride=1,
                params=wl.params(), frames=k_end - lo,
                desc=dict(workload=f"C3: long scene, {frames_per_gpu} frames/GPU (rho=4, ~{4 * frames_per_gpu // 1000}k"
                                   f" points), 6 models M=30, W=60, stride 1, T=10"))


# --------------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock, power and clock-event reasons sampled in-process through NVML
    (nvidia_ml_py) every 500 ms while the timed region runs.  (A polling nvidia-smi
    subprocess intermittently stalled the GPU work by 100-1000 ms.)"""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4}

    def __init__(self, gpu_index):
        import threading

        self.rows, self.stop_flag, self.t = [], False, None
        self.nv = None
        self.active = False  # samples are kept only between begin() and stop()
        if os.environ.get("HGM_NO_CLOCKS"):  # diagnosis only: no sampling at all
            return
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(int(gpu_index))
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None
            return

        def run():
            import time as _t

            while not self.stop_flag:
                try:
                    sm = self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM)
                    pw = self.nv.nvmlDeviceGetPowerUsage(self.h) / 1000.0
                    rs = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                    if self.active:
                        self.rows.append((sm, pw, rs))
                except Exception:
                    pass
                _t.sleep(0.5)

        self.t = threading.Thread(target=run, daemon=True)
        self.t.start()

    def begin(self):
        self.active = True

    def stop(self):
        self.active = False
        self.stop_flag = True
        if self.t is not None:
            self.t.join(timeout=2)
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        reasons = sorted({n for _, _, r in self.rows for n, bit in self.REASONS.items() if r & bit})
        return {"sm_mhz": statistics.median(r[0] for r in self.rows), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.rows),
                "power_w_max": max(r[1] for r in self.rows), "source": "NVML, 500 ms"}


# --------------------------------------------------------------------- oracle
def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name:"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def oracle_sample_rate(wl, target_s, seed=0, max_pairs=4096, threads=None):
    """Time the CPU oracle (as it stands) on a bounded random sample of pairs, on
    `threads` host threads (default: every core).  Also counts the sample's real-triple
    candidates (work.py, exact) for a candidates/s figure."""
    import oracle
    from paper_1505_00581_b200.work import count_work

    ncores = threads or os.cpu_count() or 1
    models = [oracle.model_nodes(m) for m in wl["models"]]
    order, scene = oracle.scene_nodes(wl["scene"])
    rng = np.random.default_rng(seed)
    per_off = count_work(wl["scene"].frame, wl["first"], wl["stride"], wl["count"], wl["window"],
                         wl["params"]["T"], per_offset=True)

    def run(n):
        ks = rng.integers(0, wl["count"], n)
        ms = rng.integers(0, len(models), n)
        wins = [oracle.window_range(scene.t, wl["first"] + int(k) * wl["stride"], wl["window"]) for k in ks]
        t0 = time.perf_counter()
        E, _, A, z = oracle.match_batch(models, scene, wl["params"], ms, [w[0] for w in wins], [w[1] for w in wins],
                                        ncores)
        dt = time.perf_counter() - t0
        cand = sum(int(per_off[k]) * max(models[m].n - 2, 0) for m, k in zip(ms.tolist(), ks.tolist()))
        return dt, list(zip(ms.tolist(), ks.tolist())), E, A, z, cand

    dt, _, _, _, _, _ = run(ncores)
    rate = ncores / max(dt, 1e-6)
    n = int(min(max(ncores, rate * target_s), max_pairs))
    dt, pairs, E, A, z, cand = run(n)
    return dict(value=n / dt, unit="pairs/s", cores=ncores, kind="oracle", elapsed_s=dt, pairs=pairs, E=E, A=A, z=z,
                candidates_per_s=cand / dt,
                sample=f"{n} uniformly drawn (model, offset) pairs of rank 0's workload, seed {seed}, "
                       f"fp64 C oracle, {ncores} threads")


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    wl = rank_workload(args.workload, 0, 1, args.frames_per_gpu)
    for _ in range(args.warmup):
        oracle_sample_rate(wl, 1.0, seed=99)
    vals, secs = [], []
    for s in range(args.steps):
        r = oracle_sample_rate(wl, max(2.0, args.cpu_seconds / 2), seed=s)
        vals.append(r["value"])
        secs.append(r["elapsed_s"])
    value = len(vals) / sum(1.0 / v for v in vals)  # harmonic mean = total pairs / total time
    cpu = dict(value=value, unit="pairs/s", cores=r["cores"], kind="oracle", sample=r["sample"])
    line = dict(impl="reference", metric=BASELINE_METRIC, value=value, unit="pairs/s", n_gpus=args.gpus,
                steps=args.steps, warmup=args.warmup, ms_per_step=1000 * sum(secs) / len(secs),
                higher_is_better=True, scaling="weak", vs_baseline=None, dtype="f64", data="synthetic",
                config=dict(wl["desc"]), cpu_baseline=cpu,
                e2e=dict(value=value, unit="pairs/s", h2d_bytes_per_step=0, d2h_bytes_per_step=0))
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------- own arm
def spawn_ranks(args):
    """`--gpus N` without a launcher: re-exec this command under torch.distributed.run
    (one process per GPU, rendezvous on 127.0.0.1) and return its exit code."""
    import socket

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")  # NCCL's init log (transport, NVLS) stays visible on stderr
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    print(f"bench.py: spawning {args.gpus} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    return subprocess.call(cmd, env=env)


def main():
    args = parse()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(spawn_ranks(args))
    if "WORLD_SIZE" in os.environ and int(os.environ["WORLD_SIZE"]) != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={os.environ['WORLD_SIZE']} (launcher mismatch)")
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist

    from paper_1505_00581_b200 import hgm
    from paper_1505_00581_b200.dist import pack_keys  # noqa: F401  (host twin of the device packing)
    from paper_1505_00581_b200.work import count_work

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    wl = rank_workload(args.workload, rank, world, args.frames_per_gpu)
    p = wl["params"]
    n_models = len(wl["models"])
    count = wl["count"]
    W, stride, first = wl["window"], wl["stride"], wl["first"]

    # inputs resident in HBM before timing
    scene_d = hgm.DevicePoints.from_host(wl["scene"], device=dev)
    models_d = [hgm.DevicePoints.from_host(m, device=dev) for m in wl["models"]]
    winner = torch.empty(count, dtype=torch.int32, device=dev)
    score = torch.empty(count, dtype=torch.float32, device=dev)
    maxn = torch.tensor([count], device=dev)
    if world > 1:
        dist.all_reduce(maxn, op=dist.ReduceOp.MAX)
    keys = torch.empty(int(maxn.item()), dtype=torch.int64, device=dev)
    gathered = [torch.empty_like(keys) for _ in range(world)]
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2

    def gather(win, sc):
        if world == 1:
            return
        keys.fill_(-1)
        keys[:count] = (sc.view(torch.int32).to(torch.int64) << 32) | win.to(torch.int64)
        dist.all_gather(gathered, keys)

    def step():
        scene = hgm.build_scene_index(scene_d, T_max=p["T"])
        models = [hgm.build_model_graph(m) for m in models_d]
        hgm.detect_actions(models, scene, p, first, stride, count, W, out=(winner, score, None))
        gather(winner, score)
        return scene, models

    # exact algorithmic work of the recursion (host count from the frame histogram)
    Ms = []
    for m in wl["models"]:
        Ms.append(len(np.unique(m.frame)))
    wk = count_work(wl["scene"].frame, first, stride, count, W, p["T"])
    steps_per_pair = sum(max(M - 2, 0) for M in Ms)
    work_cand = wk.real_candidates * steps_per_pair
    work_states = (wk.real_states + wk.eps_states) * steps_per_pair

    gpu_idx = local
    cvd = os.environ.get("CUDA_VISIBLE_DEVICES")
    if cvd:
        gpu_idx = cvd.split(",")[local]
    clocks = ClockSampler(gpu_idx)  # started before the warm-up: its first NVML queries are slow
    for w_ in range(args.warmup):
        if w_ == args.warmup - 1:
            hgm.set_profiling(True)  # the last warm-up step already runs with the event timers on
        flush.zero_()  # (first launch of torch's fill kernel loads its module lazily: not in the timed region)
        step()
    torch.cuda.synchronize()
    hgm.set_profiling(True)
    hgm.get_stats(reset=True)
    clocks.begin()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    ev0.record()
    dbg = os.environ.get("HGM_BENCH_DEBUG")
    evs = []
    for _ in range(args.steps):
        flush.zero_()  # L2 flush between steps (counted inside the timed region)
        step()
        if dbg:
            evs.append(torch.cuda.Event(enable_timing=True))
            evs[-1].record()
            torch.cuda.synchronize()
            st_ = hgm.get_stats(reset=False)
            print("  cumulative kernel ms:", {k: round(v, 1) for k, v in st_["ms"].items() if v}, file=sys.stderr)
    ev1.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    wall = time.perf_counter() - t0
    ms = ev0.elapsed_time(ev1)
    if dbg:
        marks = [ev0] + evs
        print("per-step ms:", [round(marks[j].elapsed_time(marks[j + 1]), 1) for j in range(len(evs))], file=sys.stderr)
    ck = clocks.stop()
    st = hgm.get_stats(reset=True)
    hgm.set_profiling(False)
    t = torch.tensor([ms, float(count * n_models), float(wl["frames"])], dtype=torch.float64, device=dev)
    if world > 1:
        tmax = t.clone()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        tsum = t.clone()
        dist.all_reduce(tsum, op=dist.ReduceOp.SUM)
        ms_max, pairs_tot, frames_tot = tmax[0].item(), tsum[1].item(), tsum[2].item()
    else:
        ms_max, pairs_tot, frames_tot = ms, float(count * n_models), float(wl["frames"])
    ms_step = ms_max / args.steps
    value = pairs_tot / (ms_step / 1000.0)
    launches = int(sum(st["launches"].values()))

    # roofline of the dominant kernel (K-DP), ALU-bound
    dp_ms = st["ms"]["dp"] / args.steps
    f_mhz = ck["sm_mhz"] or 1965.0
    # % of roofline = (10.5 N_rrr + 2 N_states) / (t x 18,944 x f_SM); expressed in
    # candidate-equivalents (the per-state FADD + min counted as 2/10.5 of a candidate)
    cand_eq = work_cand + 2.0 * work_states / ISSUE_SLOTS_PER_CAND
    achieved = cand_eq / (dp_ms / 1000.0) / 1e9  # G candidate-equivalents / s
    peak = LANES_PER_CLK * f_mhz * 1e6 / ISSUE_SLOTS_PER_CAND / 1e9
    xu_peak = XU_LANES_PER_CLK * f_mhz * 1e6 / 1e9  # G model-candidates / s (one MUFU.SQRT each)
    cand_rate = work_cand / (dp_ms / 1000.0) / 1e9
    traffic, traffic_src = None, None
    tpath = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "dp_traffic.json")
    if os.path.exists(tpath):  # DRAM bytes per K-DP launch from the committed ncu --set full capture
        with open(tpath) as fh:
            tj = json.load(fh)
        traffic, traffic_src = tj.get("dram_bytes_per_launch"), tj.get("source")
    roof = dict(bound="alu", achieved=achieved, peak=peak, unit="Gcand/s", frac=achieved / peak, traffic=traffic,
                achieved_basis="(real-triple candidates + 2/10.5 x states) / K-DP device time (SURVEY §8(d) formula)",
                candidates_per_s_g=cand_rate, frac_candidates_only=cand_rate / peak,
                traffic_unit="DRAM bytes per K-DP launch", traffic_source=traffic_src,
                xu_peak=xu_peak, xu_frac=cand_rate / xu_peak,
                xu_basis="one MUFU.SQRT per model-candidate; 148 SMs x 15.9 lanes/clk (measured) x SM clock",
                kernel="k_dp_fused", dp_ms_per_step=dp_ms, dp_share_of_step=dp_ms / ms_step,
                candidates_per_step=work_cand, states_per_step=work_states,
                peak_basis=f"148 SMs x 128 lanes x {f_mhz:.0f} MHz (median SM clock sampled in the timed region)"
                           f" / {ISSUE_SLOTS_PER_CAND} issue slots per real-triple candidate",
                kernel_ms={k: v / args.steps for k, v in st["ms"].items()})

    # e2e through the host API: pinned host inputs in, winners + scores out
    e2e = None
    if not args.no_e2e:
        def pin(a):
            t_ = torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
            return t_.numpy()

        class HP:
            pass

        def pinned(pts):
            h = HP()
            h.frame, h.x, h.y, h.saliency, h.feat = (pin(pts.frame), pin(pts.x), pin(pts.y), pin(pts.saliency),
                                                     pin(pts.feat))
            h.id = None
            return h

        sc_h = pinned(wl["scene"])
        md_h = [pinned(m) for m in wl["models"]]
        win_h = torch.empty(count, dtype=torch.int32).pin_memory().numpy()
        sco_h = torch.empty(count, dtype=torch.float32).pin_memory().numpy()
        h2d = sum(a.nbytes for a in (sc_h.frame, sc_h.x, sc_h.y, sc_h.saliency, sc_h.feat)) + sum(
            a.nbytes for m in md_h for a in (m.frame, m.x, m.y, m.saliency, m.feat))
        d2h = win_h.nbytes + sco_h.nbytes

        def step_e2e():
            scene = hgm.build_scene_index(sc_h, device=local, T_max=p["T"])
            models = [hgm.build_model_graph(m, device=local) for m in md_h]
            hgm.detect_actions(models, scene, p, first, stride, count, W, out=(win_h, sco_h, None))
            if world > 1:
                gather(torch.from_numpy(win_h).to(dev), torch.from_numpy(sco_h).to(dev))
                torch.cuda.synchronize()
            return scene, models

        for _ in range(max(2, min(args.warmup, 3))):
            step_e2e()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        ne = max(1, args.steps)
        eev = []
        for _ in range(ne):
            flush.zero_()
            step_e2e()
            if dbg:
                eev.append(torch.cuda.Event(enable_timing=True))
                eev[-1].record()
        e1.record()
        if dbg:
            torch.cuda.synchronize()
            marks = [e0] + eev
            print("e2e per-step ms:", [round(marks[j].elapsed_time(marks[j + 1]), 1) for j in range(len(eev))],
                  file=sys.stderr)
        torch.cuda.synchronize()
        me = torch.tensor([e0.elapsed_time(e1) / ne], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(me, op=dist.ReduceOp.MAX)
        e2e = dict(value=pairs_tot / (me.item() / 1000.0), unit="pairs/s", h2d_bytes_per_step=int(h2d),
                   d2h_bytes_per_step=int(d2h), ms_per_step=me.item(), steps=ne)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        r = oracle_sample_rate(wl, args.cpu_seconds)
        # parity spot-check of the timed configuration on the sampled pairs: detect's E of
        # every sampled pair, and each model's assignments (match_model_at_offsets) against
        # the oracle's z, a differing z accepted only under the near-tie rule
        from tests._parity import Checker

        models = [hgm.build_model_graph(m) for m in models_d]
        scene = hgm.build_scene_index(scene_d, T_max=p["T"])
        det = hgm.detect_actions(models, scene, p, first, stride, count, W, want_E_all=True)
        Eg = det.E_all.cpu().numpy()
        errs = [abs(float(Eg[m, k]) - e) / (1e-6 + 1e-5 * abs(e)) for (m, k), e in zip(r["pairs"], r["E"])]
        chk = Checker(wl["models"], wl["scene"], p, first, stride, W)
        ids = wl["scene"].ids()[chk.order]
        per_model = {}
        z_bad, z_ties, z_eq = [], 0, 0
        for j, (m, k) in enumerate(r["pairs"]):
            if m not in per_model:
                rm = hgm.match_model_at_offsets(models[m], scene, p, first, stride, count, W, device_out=False)
                per_model[m] = rm
            rm = per_model[m]
            zo = np.where(r["z"][j] >= 0, ids[np.maximum(r["z"][j], 0)], -1)
            msg = chk.check_pair(m, k, rm.E[k], rm.A[k], rm.z[k], r["E"][j], r["A"][j], zo)
            if msg is None:
                z_eq += 1
            elif msg == "TIE":
                z_ties += 1
            else:
                z_bad.append(msg)
        r1 = oracle_sample_rate(wl, max(3.0, args.cpu_seconds / 4), seed=1, threads=1)
        cpu = dict(value=r["value"], unit="pairs/s", cores=r["cores"], kind="oracle", sample=r["sample"],
                   cpu_model=cpu_model(), candidates_per_s=r["candidates_per_s"],
                   frames_per_s_extrapolated=r["value"] / n_models * stride,
                   frames_per_s_note="extrapolated: pairs/s / models x stride (every offset matches every model)",
                   single_thread=dict(value=r1["value"], unit="pairs/s", candidates_per_s=r1["candidates_per_s"],
                                      frames_per_s_extrapolated=r1["value"] / n_models * stride,
                                      sample=r1["sample"]),
                   parity_max_err_over_tol=max(errs) if errs else None,
                   parity_z=dict(pairs=len(r["pairs"]), identical=z_eq, near_ties=z_ties, failures=len(z_bad),
                                 first_failure=z_bad[0] if z_bad else None))

    if rank == 0:
        line = dict(metric=BASELINE_METRIC, value=value, unit="pairs/s", n_gpus=world, steps=args.steps,
                    warmup=args.warmup, ms_per_step=ms_step, higher_is_better=True, scaling="weak",
                    vs_baseline=None, dtype="f32", data="synthetic",
                    frames_per_s=frames_tot / (ms_step / 1000.0),
                    config=dict(wl["desc"], n_models=n_models, offsets_per_gpu=count, pairs_total=int(pairs_tot),
                                l2="256 MiB buffer written between timed steps (counted)",
                                parallelism=f"offset-range sharding, {world} rank(s), 1 GPU each"),
                    roofline=roof, cpu_baseline=cpu, e2e=e2e, clocks=ck, gpu_launches=launches,
                    wall_s=wall)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
