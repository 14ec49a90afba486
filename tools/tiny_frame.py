import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import golden_io as G
from paper_1905_06700_b200.rt3d import Session
name = sys.argv[1] if len(sys.argv) > 1 else "small_s3"
sc, cfg, _ = G.scene(name)
cfg.max_iters = 10
with Session(0) as s:
    s.set_scene(sc)
    for _ in range(2):
        s.reconstruct_async(cfg)
    s.synchronize()
    print(s.report()["total_seconds"])
