"""Phase timings of small frames (fixed per-phase overhead)."""
import sys, json
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import golden_io as G
from paper_1905_06700_b200.rt3d import Session
for name in sys.argv[1:] or ["small_s3", "dense_12"]:
    sc, cfg, _ = G.scene(name)
    cfg.max_iters = 10
    with Session(0) as s:
        s.set_scene(sc)
        for _ in range(3):
            s.reconstruct_async(cfg)
        s.synchronize()
        s.profile(True)
        s.reconstruct_async(cfg)
        s.synchronize()
        ph = {}
        for n, ns in s.profile_phases():
            d = ph.setdefault(n, [0, 0.0]); d[0] += 1; d[1] += ns / 1e3
        rep = s.report()
        print(name, "pix", sc.n_pixels, "pts", rep["points"], "total ms", round(rep["total_seconds"] * 1e3, 3))
        print("  per-call us:", {k: round(v[1] / v[0], 2) for k, v in ph.items()})
