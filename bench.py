#!/usr/bin/env python3
"""RT3D frame benchmark (BASELINE.json metric: frames/s and ms/frame).

Workload (BASELINE.json configs[1]): a synthetic
141x141-pixel, 4613-bin "polystyrene head" frame (back plane with a hole +
head bump, 3 signal photons/px, SBR 13), reconstructed with the acceptance
preset at apss_radius 0.02 m, 25 PALM iterations, stop_tol 0.  One step =
one frame through splidar::reconstruct's device replacement.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]

Ours: inputs resident in HBM, one persistent kernel per frame, each frame
timed with CUDA events on the session stream, the 126 MB L2 flushed between
frames.  e2e: the same frames through the C ABI from pinned host buffers
(cube upload + reconstruct + cloud/background download), wall clock.
N > 1 (torchrun): frames are independent, each rank reconstructs its own
stream of frames (weak scaling, no collective on the data path).
--impl reference: the reference CPU implementation (the headers compiled
unchanged, oracle/_ref/libref.so) on the host cores, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

sys.path.insert(0, str(ROOT / "tools"))
import workloads  # noqa: E402

PAPER_MS_PER_FRAME = 13.0  # 141x141x4613 on a Titan Xp


def config_b():
    """141x141 px, 4613 bins of 0.3 mm."""
    name, spec, seed, cfg = workloads.config_b()
    return spec, seed, cfg, name


def shared_config(spec, cfg, n_events) -> dict:
    """The `config` object both arms print (identical keys and values)."""
    return {"workload": workloads.config_b()[0], "pixels": spec.rows * spec.cols,
            "bins": spec.bins, "palm_iterations": cfg.max_iters, "events": int(n_events),
            "recon": "acceptance preset, apss_radius 0.02 m, stop_tol 0 (fixed budget)",
            "l2": "GPU arm: flushed between frames (256 MB write)"}


KERNEL_NAMES = {
    "stage_first": "rt3d::stage_kernel<ST_FIRST> (init peaks, spawn, first nll+grad sweep, depth block 0)",
    "stage_depth": "rt3d::stage_kernel<ST_DEPTH> (depth candidates + backtracking)",
    "apss": "rt3d::apss_kernel (APSS ball moments, warp per point)",
    "apss_fit": "rt3d::apss_fit_kernel (sphere fit, projection, pinning)",
    "iteration": "rt3d::stage_kernel<ST_ITER> (one PALM iteration: APSS moments + fit, intensity block, "
                 "kNN, prune, background block, nll, next depth block)",
    "stage_intensity": "rt3d::stage_kernel<ST_INTENSITY> (intensity grad + candidates)",
    "knn": "rt3d::knn_kernel (kNN intensity filter)",
    "stage_tail": "rt3d::stage_kernel<ST_TAIL> (prune, background block, nll, next depth block)",
}


def class_bytes(sc, rep, fused_depth: bool = True) -> dict:
    """Algorithmic HBM bytes of one frame per kernel class (DESIGN.md §4,
    SURVEY.md §8d): every likelihood sweep reads the CSR cube (8 B/event),
    per-pixel offsets/bucket/background/gain/dead (29 B/px) and t, r, bucket
    index (20 B/point); gradient sweeps write grad+curv (16 B/unit),
    candidate sweeps write the candidate (8 B/unit); APSS 17 B/pt, kNN
    24 B/pt, prune 9 B/pt in + 33 B/survivor + 4 B/px; init 8E + 29 Npix +
    33 P0."""
    E, npix = len(sc.events), sc.n_pixels
    steps = rep["steps"]

    def sweep(P, extra):
        return 8.0 * E + 29.0 * npix + 20.0 * P + extra

    b = dict.fromkeys(KERNEL_NAMES, 0.0)
    P0 = int(steps[0]["points_before"]) if len(steps) else 0
    b["stage_first"] = 8.0 * E + 29.0 * npix + 33.0 * P0 + sweep(P0, 16.0 * P0)
    for k, st in enumerate(steps):
        P, P1 = int(st["points_before"]), int(st["points_after"])
        if P > 0:
            # the depth block runs at the end of the kernel that computed its
            # gradients (ST_FIRST for iteration 0, else the previous ST_TAIL)
            dk = "stage_depth" if not fused_depth else ("stage_first" if k == 0 else "stage_tail")
            b[dk] += (1 + int(st["depth_backtracks"])) * sweep(P, 8.0 * P)
            b["apss"] += 8.0 * P          # t in (neighbours are L2/SMEM reuse)
            b["apss_fit"] += 9.0 * P      # t out + flags
            b["stage_intensity"] += sweep(P, 16.0 * P) + \
                (1 + int(st["intensity_backtracks"])) * sweep(P, 8.0 * P)
            b["knn"] += 24.0 * P
            b["stage_tail"] += 9.0 * P + 33.0 * P1 + 4.0 * npix
        b["stage_tail"] += sweep(P1, 16.0 * npix) + \
            (1 + int(st["background_backtracks"])) * sweep(P1, 8.0 * npix) + \
            sweep(P1, 16.0 * P1)   # nll after the iteration fused with the next grad_t
    return b


def frame_bytes(sc, rep) -> float:
    return sum(class_bytes(sc, rep).values())


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4)
                          if len(r) > 5 + k and r[5 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def dist_init():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def barrier_max(value: float, world: int, device: int) -> float:
    if world == 1:
        return value
    import torch
    import torch.distributed as dist
    t = torch.tensor([value], dtype=torch.float64, device=f"cuda:{device}")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world: int):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def load_measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def apss_fp64(points, radius: float, us_per_launch: float, frames: int = 1,
              peak_tflops: float = None):
    """The APSS kernel against the FP64 roof: ~70 flop per
    (point, neighbour) pair for distance, weight, mean, covariance and the
    Pratt moments, plus ~3000 flop per point for the 3x3 and 5x5 eigensolves.
    Neighbour counts come from the final cloud (ball of `radius`, self
    included) of the first frame, times the frames one launch processes, so
    this is an estimate of one launch's flops."""
    try:
        from scipy.spatial import cKDTree
    except ImportError:
        return None
    if len(points) == 0 or not us_per_launch:
        return None
    xyz = np.stack([points["x"], points["y"], points["z"]], axis=1)
    nbrs = cKDTree(xyz).query_ball_point(xyz, radius, return_length=True)
    flops = frames * (70.0 * float(np.sum(nbrs)) + 3000.0 * len(points))
    achieved = flops / (us_per_launch * 1e-6) / 1e12
    return {"achieved": achieved, "unit": "TFLOP/s", "peak": peak_tflops,
            "frac": achieved / peak_tflops, "flops_per_launch": flops,
            "mean_neighbours": float(np.mean(nbrs)),
            "peak_source": "measured in this run: rt3d_measure_fp64_peak (DFMA chains, "
                           "full device, best of 5)",
            "note": "APSS is FP64-issue-bound; its HBM fraction is ~0 because its working "
                    "set stays in L2"}


def ncu_traffic_per_launch(cls: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of a kernel
    class, from the committed `ncu --set full` capture summary."""
    p = ROOT / "profiles" / "ncu_traffic.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())[cls]["dram_bytes_per_launch"])
        except Exception:
            return None
    return None


def reference_frame(sc, cfg, threads: int = 0):
    """The reference implementation itself (headers compiled unchanged,
    oracle/_ref/libref.so) timed on the host cores with steady_clock around
    splidar::reconstruct (the bench_scaling method, eval.hpp:229-233); else
    the C port.  Returns (seconds, kind, cores, cloud)."""
    import ctypes as C
    sys.path.insert(0, str(ROOT / "tests"))
    import oracle_lib as O
    from paper_1905_06700_b200.abi import POINT_DTYPE, Point, ptr
    if O.ref_available():
        lib = O.ref()
        lib.ref_set_threads(threads)
        n, it, secs = C.c_uint64(), C.c_int(), C.c_double()
        rc = lib.ref_reconstruct(C.byref(sc.cube_c()), C.byref(sc.sensor_c()),
                                 C.byref(cfg.to_c()), C.byref(n), C.byref(it), C.byref(secs))
        if rc != 0:
            raise RuntimeError(lib.ref_last_error().decode())
        cloud = np.zeros(max(n.value, 1), POINT_DTYPE)
        lib.ref_result_copy(ptr(cloud, Point), None)
        cores = threads if threads > 0 else (os.cpu_count() or 1)
        return secs.value, "reference", cores, cloud[: n.value]
    t0 = time.perf_counter()
    r = O.reconstruct(sc, cfg, "oracle")
    return time.perf_counter() - t0, "port", 1, r["points"]


def reference_cube(spec, seed):
    """The workload's cube from the reference's own simulate_cube
    (simulate.hpp:139-223, oracle/_ref/libref.so) on the SceneSpec text."""
    sys.path.insert(0, str(ROOT / "tests"))
    import oracle_lib as O
    if O.ref_available():
        return O.ref_simulate(workloads.spec_text(spec), seed)
    from scenegen.scene import simulate
    return simulate(spec, seed)


def run_reference_arm(args, world, rank):
    if rank != 0:
        return 0
    spec, seed, cfg, workload = config_b()
    sc = reference_cube(spec, seed)
    times = []
    for k in range(args.warmup + args.steps):
        secs, kind, cores, _ = reference_frame(sc, cfg)
        if k >= args.warmup:
            times.append(secs)
    total = sum(times)
    fps = len(times) / total
    line = {
        "impl": "reference", "metric": "frames/s", "value": fps, "unit": "frames/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / len(times), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": shared_config(spec, cfg, len(sc.events)),
        "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": cores, "kind": kind,
                         "sample": f"{len(times)} full frames (25 PALM iterations) after "
                                   f"{args.warmup} warm-up frames; cube from the reference's "
                                   "own simulate_cube"},
        "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def large_array_leg(local: int, frames: int = 3) -> dict:
    """Config E (1024x1024 px x 2048 bins, ~68M events, 548 MB
    of CSR events, HBM-resident) on one GPU: ms/frame, and per kernel class
    the algorithmic bytes per launch (class_bytes) over the CUDA-event launch
    time.  The likelihood sweeps (stage kernels) are the north star's
    'gradient kernels' measured where HBM binds."""
    import torch
    from paper_1905_06700_b200.rt3d import Session
    from scenegen.scene import simulate
    name, spec, seed, cfg = workloads.config_e()
    t0 = time.perf_counter()
    sc = simulate(spec, seed)
    sim_s = time.perf_counter() - t0
    out = {"workload": name, "pixels": sc.n_pixels, "bins": sc.n_bins,
           "events": int(len(sc.events)), "event_bytes": int(len(sc.events)) * 8,
           "palm_iterations": cfg.max_iters, "host_simulate_s": sim_s}
    with Session(local) as s:
        s.set_scene(sc)
        s.reconstruct_async(cfg)
        s.synchronize()
        stream = torch.cuda.ExternalStream(s.stream_ptr, device=torch.device("cuda", local))
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(frames)]
        with torch.cuda.stream(stream):
            for a, b in evs:
                a.record(stream)
                s.reconstruct_async(cfg)
                b.record(stream)
        stream.synchronize()
        ms = [a.elapsed_time(b) for a, b in evs]
        rep = s.report()
        s.time_kernels(True)
        s.reconstruct_async(cfg)
        kt = s.kernel_times()
        s.time_kernels(False)
    cb = class_bytes(sc, rep, fused_depth=kt["stage_depth"][1] == 0)
    peak, src = load_measured_peaks()
    classes = {}
    for cls, (kms, n) in kt.items():
        if not n:
            continue
        per = cb[cls] / n
        gbs = per / (kms / n) / 1e6
        classes[cls] = {"ms_per_frame": kms, "launches": n, "us_per_launch": 1e3 * kms / n,
                        "algorithmic_bytes_per_launch": per, "gbs": gbs, "hbm_frac": gbs / peak}
    out.update({"ms_per_frame": statistics.mean(ms), "frames_per_s": 1e3 / statistics.mean(ms),
                "points_final": int(rep["points"]), "kernel_classes": classes,
                "sweep_roofline": {"kernel": KERNEL_NAMES["stage_tail"], "bound": "hbm",
                                   "achieved": classes["stage_tail"]["gbs"], "peak": peak,
                                   "unit": "GB/s", "frac": classes["stage_tail"]["hbm_frac"],
                                   "peak_source": src},
                "note": "frames measured with CUDA events on the session stream, inputs "
                        "resident; the working set (548 MB of events) exceeds L2"})
    return out


def parity_block(sess, sc, cfg, ref_cloud, gpu_cloud) -> dict:
    """bench-time parity at the benchmarked workload (tests/parity.py): the
    GPU cloud of the timed frames against the reference's own cloud from the
    cpu_baseline run (free running, reported), every PALM step against the
    reference from its own state (asserted by the tests), and the full
    reconstruction against the C oracle (same trajectory)."""
    sys.path.insert(0, str(ROOT / "tests"))
    import oracle_lib as O
    import parity as PY
    out = {"tolerance": {"t_bins": PY.T_TOL_BINS, "r_rel": PY.R_TOL_REL, "count_rel": PY.COUNT_TOL}}
    if ref_cloud is not None:
        out["vs_reference_free_running"] = PY.cloud_diff(gpu_cloud, ref_cloud)
    if O.ref_available():
        out["init_bitexact_vs_reference"] = PY.init_bitexact(sess, sc, cfg, "ref")
        w = PY.stepwise(sess, sc, cfg, "ref")
        w["within_tolerance"] = bool(w["same_cells"] and w["count_rel"] <= PY.COUNT_TOL and
                                     w["max_dt_bins"] <= PY.T_TOL_BINS and
                                     w["max_rel_dr"] <= PY.R_TOL_REL)
        out["vs_reference_stepwise"] = w
    t0 = time.perf_counter()
    d = PY.free_running(sess, sc, cfg, "oracle")
    d["within_tolerance"] = PY.within_tolerance(d)
    d["oracle_seconds"] = time.perf_counter() - t0
    out["vs_oracle_free_running"] = d
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--e2e-groups", type=int, default=2, choices=[1, 2],
                    help="e2e session groups: 1 = one group, copies between batches; "
                         "2 = two groups alternating batches (rt3d_session_after orders the "
                         "batches on the device), one group's copies overlapping the other's "
                         "frames")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--no-large", action="store_true", help="skip the config-E leg")
    ap.add_argument("--batch", type=int, default=20,
                    help="frames per step (rt3d_reconstruct_batch), 1..32")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    world, rank, local = dist_init()
    if args.impl == "reference":
        rc = run_reference_arm(args, world, rank)
        barrier(world)
        return rc

    import torch
    from paper_1905_06700_b200.abi import POINT_DTYPE
    from paper_1905_06700_b200.rt3d import Session
    from scenegen.scene import simulate

    torch.cuda.set_device(local)
    spec, seed, cfg, workload = config_b()
    NB = args.batch
    # a stream of NB frames of the scene (photon noise seeds seed .. seed+NB-1)
    cubes = [simulate(spec, seed + k) for k in range(NB)]
    sc = cubes[0]
    sessions = [Session(local) for _ in range(NB)]
    for s, c in zip(sessions, cubes):
        s.set_scene(c)
    sess = sessions[0]
    stream = torch.cuda.ExternalStream(sess.stream_ptr, device=torch.device("cuda", local))
    flush = torch.empty(64 * 2 ** 20, dtype=torch.float32, device=f"cuda:{local}")  # 256 MB > L2

    def run_batch():
        Session.reconstruct_batch_async(sessions, cfg)

    # warm-up (module load, buffers, CUDA graphs)
    for _ in range(args.warmup):
        run_batch()
        sess.reconstruct_async(cfg)
    sess.synchronize()

    def timed(fn, K):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(K)]
        with torch.cuda.stream(stream):
            for k in range(K):
                flush.zero_()  # evict the working set from L2 between steps
                evs[k][0].record(stream)
                fn()
                evs[k][1].record(stream)
        stream.synchronize()
        return [x.elapsed_time(y) for x, y in evs]

    K = args.steps
    barrier(world)
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        t_wall0 = time.perf_counter()
        step_ms = timed(run_batch, K)           # one step = one batch of NB frames
        torch.cuda.synchronize()
        t_wall = time.perf_counter() - t_wall0
    barrier(world)
    # single-frame latency (one frame per launch sequence), reported alongside
    single_ms = timed(lambda: sess.reconstruct_async(cfg), K)
    # per-kernel breakdown: CUDA events around every launch of a batch on the
    # launching stream (the value pass replays each batch as one CUDA graph,
    # inside which events cannot time kernels)
    sess.time_kernels(True)
    torch.cuda.synchronize()
    timed_ms = timed(run_batch, K)
    ktimes = sess.kernel_times()
    sess.time_kernels(False)
    fp64_peak = sess.measure_fp64_peak()
    dev_s = sum(step_ms) / 1e3
    dev_s_max = barrier_max(dev_s, world, local)
    value = world * K * NB / dev_s_max
    rep = sess.report()
    pts, _ = sess.state()

    # e2e through the public API from pinned host buffers: every step uploads
    # its NB cubes (rt3d_set_cube), reconstructs them as one batch
    # (rt3d_reconstruct_batch) and downloads every cloud and background
    # (rt3d_state_copy), all inside the timed region.  Two groups of sessions
    # (full-size grids) alternate: rt3d_session_after queues each batch behind
    # the other group's previous batch on the device, so the frames run one
    # after another while one group's copies overlap the other's frames.
    import copy
    n_e2e = args.e2e_steps or max(K // 2, 6)
    pinned = []
    for c in cubes:
        cp = copy.copy(c)
        off = torch.empty(len(c.offsets), dtype=torch.int64, pin_memory=True).numpy().view(np.uint64)
        ev = torch.empty(len(c.events) * 2, dtype=torch.int32,
                         pin_memory=True).numpy().view(c.events.dtype)
        off[:] = c.offsets
        ev[:] = c.events
        cp.offsets, cp.events = off, ev
        pinned.append(cp)
    P_cap = cfg.init_max_returns * spec.superres * spec.superres * sc.n_pixels
    outs = [(torch.empty(P_cap * 64, dtype=torch.uint8, pin_memory=True).numpy().view(POINT_DTYPE),
             torch.empty(sc.n_pixels, dtype=torch.float64, pin_memory=True).numpy())
            for _ in range(NB)]
    import ctypes as C
    from paper_1905_06700_b200 import rt3d as R
    two = args.e2e_groups == 2
    group_b = [Session(local) for _ in range(NB)] if two else []
    for s, c in zip(group_b, cubes):
        s.set_scene(c)
    groups = [sessions, group_b] if two else [sessions, sessions]

    def upload_launch(g):
        for s, c in zip(g, pinned):
            s.set_cube(c)
        if two:
            g[0].after(groups[1][0] if g is groups[0] else groups[0][0])
        Session.reconstruct_batch_async(g, cfg)

    def download(g):
        d2h = 0
        for s, (op, ob) in zip(g, outs):
            n = R._u64()
            R._check(R.lib().rt3d_state_size(s.h, C.byref(n)))
            R._check(R.lib().rt3d_state_copy(s.h, R.ptr(op, R.Point), R.ptr(ob, R._dbl)))
            d2h += n.value * 64 + ob.nbytes
        return d2h

    upload_launch(groups[0])
    download(groups[0])
    if two:
        upload_launch(groups[1])
        download(groups[1])
    barrier(world)
    t0 = time.perf_counter()
    if two:
        upload_launch(groups[0])
        for k in range(n_e2e):
            if k + 1 < n_e2e:
                upload_launch(groups[(k + 1) % 2])  # runs while batch k finishes
            d2h = download(groups[k % 2])
    else:
        for k in range(n_e2e):  # full grids; each step's copies around its batch
            upload_launch(groups[0])
            d2h = download(groups[0])
    e2e_s = time.perf_counter() - t0
    e2e_s = barrier_max(e2e_s, world, local)
    e2e_fps = world * n_e2e * NB / e2e_s
    h2d = sum(c.offsets.nbytes + c.events.nbytes for c in cubes)
    if two:
        for s in sessions:
            s.set_sharing(1)
    for s in group_b:
        s.close()

    peak, peak_src = load_measured_peaks()
    # algorithmic bytes of one batch: every frame's own report
    cb = dict.fromkeys(KERNEL_NAMES, 0.0)
    for s, c in zip(sessions, cubes):
        for k, v in class_bytes(c, s.report(), fused_depth=ktimes["stage_depth"][1] == 0).items():
            cb[k] += v
    if ktimes["iteration"][1] > 0:  # one launch per iteration: its classes merge
        for c in ("apss", "apss_fit", "stage_intensity", "knn", "stage_tail"):
            cb["iteration"] += cb[c]
            cb[c] = 0.0
    fb = sum(cb.values())
    classes = {}
    for cls, (ms, n) in ktimes.items():
        per_launch_bytes = cb[cls] * K / n if n else 0.0
        classes[cls] = {"ms_per_frame": ms / (K * NB), "launches_per_batch": n / K,
                        "us_per_launch": 1e3 * ms / n if n else None,
                        "algorithmic_bytes_per_launch": per_launch_bytes,
                        "gbs": per_launch_bytes / (ms / n) / 1e6 if n and ms else None}
    dom = max(classes, key=lambda c: classes[c]["ms_per_frame"])
    dc = classes[dom]
    achieved = dc["gbs"]
    launches = sum(n for _, n in ktimes.values())

    cpu = None
    parity = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        secs, kind, cores, ref_cloud = reference_frame(sc, cfg)
        cpu = {"value": 1.0 / secs, "unit": "frames/s", "cores": cores, "kind": kind,
               "sample": "1 full frame of the same workload (25 PALM iterations), "
                         "reference headers compiled unchanged (oracle/_ref), all host threads"}
        if not args.no_parity:
            parity = parity_block(sess, sc, cfg, ref_cloud, pts)
    large = None
    if rank == 0 and world == 1 and not args.no_large:
        large = large_array_leg(local)

    if rank == 0:
        line = {
            "metric": "frames/s", "value": value, "unit": "frames/s", "n_gpus": world,
            "steps": K, "warmup": args.warmup, "ms_per_step": 1e3 * dev_s_max / K,
            "higher_is_better": True, "scaling": "weak",
            "vs_baseline": value / (1000.0 / PAPER_MS_PER_FRAME),
            "dtype": "f64", "data": "synthetic",
            "config": shared_config(spec, cfg, len(sc.events)),
            "details": {
                "frames_per_step": NB,
                "step": f"one batch of {NB} frames (photon-noise seeds {seed}..{seed + NB - 1}) "
                        "through rt3d_reconstruct_batch: one launch sequence, a frame axis "
                        "in every kernel's grid, each frame with its own controller",
                "points_init": int(rep["steps"][0]["points_before"]) if len(rep["steps"]) else 0,
                "points_final": int(rep["points"]), "parallelism": f"frames x{world} (replicas)",
                "vs_baseline_ref": "paper GPU 13 ms/frame on Titan Xp (BASELINE.md)",
                "ms_per_step_p50": statistics.median(step_ms),
                "ms_per_step_direct_launch": sum(timed_ms) / K,
                "single_frame_latency_ms_p50": statistics.median(single_ms),
                "single_frame_latency_ms_min": min(single_ms),
                "single_frame_fps": 1e3 * K / sum(single_ms),
                "frame_launch": "one CUDA graph per batch (captured once, replayed)",
            },
            "e2e": {"value": e2e_fps, "unit": "frames/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h),
                    "mode": f"public API per step: rt3d_set_cube x{NB} from pinned host cubes, "
                            f"rt3d_reconstruct_batch, rt3d_state_copy x{NB} (cloud + background) "
                            "into pinned host buffers; wall clock; "
                            + ("two session groups with full-size grids alternate batches "
                               "(rt3d_session_after orders them on the device), so one batch's "
                               "copies overlap the other's frames" if args.e2e_groups == 2 else
                               "one session group with full-size grids, each step's copies "
                               "around its batch")},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": ncu_traffic_per_launch(dom),
                         "kernel": KERNEL_NAMES[dom],
                         "share_of_step": dc["ms_per_frame"] * NB / (sum(timed_ms) / K),
                         "us_per_launch": dc["us_per_launch"],
                         "algorithmic_bytes_per_launch": dc["algorithmic_bytes_per_launch"],
                         "peak_source": peak_src,
                         "timing": "CUDA events on the launching stream around every launch, "
                                   "summed over a second timed pass of K batches launched "
                                   "directly (the value pass replays each batch as a CUDA "
                                   "graph)"},
            "frame_roofline": {"achieved": fb / (dev_s / K) / 1e9, "unit": "GB/s",
                               "algorithmic_bytes_per_step": fb},
            "kernel_classes": classes,
            "gpu_launches": launches,
            "clocks": clocks.summary(),
            "wall_s_timed_region": t_wall,
        }
        if cpu:
            line["cpu_baseline"] = cpu
        if parity:
            line["parity"] = parity
        if large:
            line["large_array"] = large
        if dom == "apss":
            # APSS keeps its working set in L2 and is bound by FP64 issue, not
            # HBM: its roofline is the FP64 one (the measured DFMA peak of
            # this device), the HBM view is kept beside it
            fp = apss_fp64(pts, cfg.apss_radius, dc["us_per_launch"], NB, fp64_peak)
            if fp:
                hbm_view = {k: line["roofline"][k] for k in
                            ("achieved", "peak", "unit", "frac", "algorithmic_bytes_per_launch",
                             "peak_source")}
                hbm_view["bound"] = "hbm"
                rf = line["roofline"]
                line["roofline"] = {
                    "bound": "fp64", "achieved": fp["achieved"], "peak": fp["peak"],
                    "unit": "TFLOP/s", "frac": fp["frac"], "traffic": rf["traffic"],
                    "kernel": rf["kernel"], "share_of_step": rf["share_of_step"],
                    "us_per_launch": rf["us_per_launch"],
                    "flops_per_launch": fp["flops_per_launch"],
                    "mean_neighbours": fp["mean_neighbours"],
                    "peak_source": fp["peak_source"],
                    "bound_note": "FP64 CUDA-core arithmetic (neither HBM nor tensor cores); "
                                  "flop model of SURVEY.md §8d: 70 flop per (point, neighbour) "
                                  "pair + 3000 per point",
                    "timing": rf["timing"], "hbm": hbm_view}
        print(json.dumps(line), flush=True)
    for s in sessions:
        s.close()
    barrier(world)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
