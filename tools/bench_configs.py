"""Frames/s on the other SURVEY.md §8d configurations (A, C; D, E on request), one stream, CUDA
events around each frame (inputs resident), plus a short-run parity check
against the C oracle (max |dt| and point counts after `check_iters`).
usage: python tools/bench_configs.py [frames] [A C D E ...]
(E, 1M pixels, skips the oracle check: the oracle needs minutes per iteration.)"""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1905_06700_b200.abi import Config  # noqa: E402
from paper_1905_06700_b200.rt3d import Session  # noqa: E402
from scenegen.scene import SceneSpec, SurfaceSpec, simulate  # noqa: E402


def config_a():
    spec = SceneSpec(rows=64, cols=64, bins=1024, bin_resolution_m=0.01, pixel_pitch_m=0.02,
                     irf_sigma_bins=1.5, target_ppp=50.0, target_sbr=1.0,
                     surfaces=[SurfaceSpec(depth_m=7.0),
                               SurfaceSpec(depth_m=5.0, region=(16, 16, 48, 48))])
    cfg = Config(max_iters=25, stop_tol=0.0, apss_radius=0.16, knn_k=9, r_min=0.25,
                 init_max_returns=3, init_peak_threshold=0.5, init_min_separation=6)
    return "A 64x64x1024 two planes, ~100 photons/px", spec, 100, cfg


def config_c(frame=0):
    s = 3
    pitch = 0.05
    n = 32 * s
    spec = SceneSpec(rows=32, cols=32, bins=153, superres=s, bin_resolution_m=0.0375,
                     pixel_pitch_m=pitch, irf_sigma_bins=1.5, target_ppp=450.0, target_sbr=1.0,
                     surfaces=[
                         SurfaceSpec(depth_m=1.5, holes=[(10, 10, 20, 20), (40, 50, 55, 70),
                                                         (70, 20, 85, 35)]),
                         SurfaceSpec(kind="bump", depth_m=3.0, bump_amp=-0.2, bump_width=0.4,
                                     bump_cx=(30 + frame) * pitch, bump_cy=48 * pitch,
                                     region=(10, 20, 80, 76)),
                         SurfaceSpec(depth_m=4.5)])
    cfg = Config(max_iters=25, stop_tol=0.0, apss_radius=0.30, knn_k=9, r_min=0.2,
                 init_max_returns=3, init_peak_threshold=0.5, init_min_separation=6)
    return "C 32x32x153 superres 3 (96x96), three surfaces, ~900 photons/px", spec, 1000 + frame, cfg


def _camouflage(n, scale):
    """a camouflage net with a grid of holes at
    5 m, a target bump at 8 m, a back plane at 12 m (<= 3 surfaces per px)."""
    pitch = 0.02
    step, hole = 16 * scale, 8 * scale
    holes = [(a, b, a + hole, b + hole) for a in range(0, n, step) for b in range(0, n, step)]
    c = n * pitch / 2
    return [SurfaceSpec(depth_m=5.0, holes=holes),
            SurfaceSpec(kind="bump", depth_m=8.0, bump_amp=-0.5, bump_cx=c, bump_cy=c,
                        bump_width=0.4 * c),
            SurfaceSpec(depth_m=12.0)]


def config_d():
    spec = SceneSpec(rows=256, cols=256, bins=2048, bin_resolution_m=0.01, pixel_pitch_m=0.02,
                     irf_sigma_bins=1.5, target_ppp=30.0, target_sbr=1.0,
                     surfaces=_camouflage(256, 1))
    return "D 256x256x2048 camouflage, ~60 photons/px", spec, 256, config_a()[3]


def config_e():
    spec = SceneSpec(rows=1024, cols=1024, bins=2048, bin_resolution_m=0.01, pixel_pitch_m=0.02,
                     irf_sigma_bins=1.5, target_ppp=50.0, target_sbr=1.0,
                     surfaces=_camouflage(1024, 4))
    return "E 1024x1024x2048 camouflage, ~100 photons/px", spec, 1024, config_a()[3]


def run(name, spec, seed, cfg, frames, check_iters=3):
    import dataclasses
    import oracle_lib as O
    sc = simulate(spec, seed)
    out = {"config": name, "pixels": sc.n_pixels, "bins": sc.n_bins, "events": int(len(sc.events))}
    with Session(0) as s:
        s.set_scene(sc)
        for _ in range(3):
            s.reconstruct_async(cfg)
        s.synchronize()
        stream = torch.cuda.ExternalStream(s.stream_ptr, device=torch.device("cuda", 0))
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(frames)]
        with torch.cuda.stream(stream):
            for k in range(frames):
                ev[k][0].record(stream)
                s.reconstruct_async(cfg)
                ev[k][1].record(stream)
        stream.synchronize()
        ms = [a.elapsed_time(b) for a, b in ev]
        rep = s.report()
        s.time_kernels(True)
        for _ in range(3):
            s.reconstruct_async(cfg)
        kt = s.kernel_times()
        s.time_kernels(False)
        out["kernel_ms_per_frame"] = {k: round(v[0] / 3, 3) for k, v in kt.items() if v[1]}
        out["backtracks_per_frame"] = {b: int(rep["steps"][f"{b}_backtracks"].sum())
                                       for b in ("depth", "intensity", "background")}
        out.update({"ms_per_frame": sum(ms) / frames, "frames_per_s": 1e3 * frames / sum(ms),
                    "points": int(rep["points"]), "iterations": int(rep["iterations"])})
        if check_iters == 0:
            return out
        short = dataclasses.replace(cfg, max_iters=check_iters)
        g = s.reconstruct(short)
        t0 = time.perf_counter()
        o = O.reconstruct(sc, short, "oracle")
        out["oracle_s"] = time.perf_counter() - t0
        same = len(g["points"]) == len(o["points"])
        out["parity_iters"] = check_iters
        out["parity_points"] = [int(len(g["points"])), int(len(o["points"]))]
        if same and len(o["points"]):
            out["parity_max_dt_bins"] = float(np.max(np.abs(g["points"]["t"] - o["points"]["t"])))
            out["parity_max_rel_dr"] = float(np.max(
                np.abs(g["points"]["intensity"] - o["points"]["intensity"]) /
                np.maximum(np.abs(o["points"]["intensity"]), 1e-300)))
    return out


def main():
    frames = int(sys.argv[1]) if len(sys.argv) > 1 else 10
    which = sys.argv[2:] or ["A", "C"]
    table = {"A": (config_a, 3), "C": (config_c, 3), "D": (config_d, 1), "E": (config_e, 0)}
    for key in which:
        make, check = table[key]
        name, spec, seed, cfg = make()
        print(json.dumps(run(name, spec, seed, cfg, frames, check)), flush=True)


if __name__ == "__main__":
    main()
