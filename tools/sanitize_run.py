"""Small workloads for compute-sanitizer (memcheck / racecheck / synccheck):
reconstruct on two golden scenes (identity and FFT background), the
operators on a golden cloud, and the streaming API.  Run as
  compute-sanitizer --tool racecheck python tools/sanitize_run.py"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import golden_io as G  # noqa: E402
from paper_1905_06700_b200.rt3d import Session  # noqa: E402

with Session(0) as s:
    for name in ("small_s3", "superres_8"):
        sc, cfg, d = G.scene(name)
        cfg.max_iters = 2
        s.set_scene(sc)
        r = s.reconstruct(cfg)
        cfg.background_mode = 1
        r2 = s.reconstruct(cfg)
        s.upload_state(d["init_points"], d["init_background"])
        s.grads()
        s.nll()
        pts = d["init_points"]
        s.apss_project(pts, cfg.apss_radius)
        s.knn_filter(pts, cfg.knn_k, cfg.apss_radius)
        s.prune(pts, 0.2)
        t = s.frame_submit(sc, cfg)
        s.frame_collect(t)
        print(name, len(r["points"]), len(r2["points"]), flush=True)
print("sanitize workload done")
