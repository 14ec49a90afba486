"""Run config-B frames (bench workload) for profiling under ncu.
usage: python tools/profile_frame.py [n_frames]"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_1905_06700_b200.rt3d import Session  # noqa: E402
from scenegen.scene import simulate  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2
spec, seed, cfg, _ = bench.config_b()
sc = simulate(spec, seed)
with Session(0) as s:
    s.set_scene(sc)
    for _ in range(n):
        s.reconstruct_async(cfg)
    s.synchronize()
    rep = s.report()
    print("frames", n, "points", rep["points"], "iters", rep["iterations"],
          "device ms", rep["total_seconds"] * 1e3)
