"""Frames/s on the other SURVEY.md §8d configurations (A, C; D, E on request), one stream, CUDA
events around each frame (inputs resident), plus a short-run parity check
against the C oracle (max |dt| and point counts after `check_iters`).
usage: python tools/bench_configs.py [frames] [A C D E ...]
(E, 1M pixels, skips the oracle check: the oracle needs minutes per iteration.)"""
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
sys.path.insert(0, str(ROOT / "tools"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1905_06700_b200.abi import Config  # noqa: E402
from paper_1905_06700_b200.rt3d import Session  # noqa: E402
from scenegen.scene import SceneSpec, SurfaceSpec, simulate  # noqa: E402


from workloads import config_a, config_b, config_c, config_d, config_e  # noqa: E402,F401


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
    table = {"A": (config_a, 3), "B": (config_b, 3), "C": (config_c, 3), "D": (config_d, 1),
             "E": (config_e, 0)}
    for key in which:
        make, check = table[key]
        name, spec, seed, cfg = make()
        if os.environ.get("CHECK_ITERS"):
            check = int(os.environ["CHECK_ITERS"])
        print(json.dumps(run(name, spec, seed, cfg, frames, check)), flush=True)


if __name__ == "__main__":
    main()
