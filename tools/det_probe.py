"""Run config-B frames repeatedly; report whether outputs are bitwise identical."""
import sys, hashlib
sys.path.insert(0, '.')
import bench
from paper_1905_06700_b200.rt3d import Session
from scenegen.scene import simulate
spec, seed, cfg, _ = bench.config_b()
cfg.max_iters = int(sys.argv[1]) if len(sys.argv) > 1 else 25
n = int(sys.argv[2]) if len(sys.argv) > 2 else 6
sc = simulate(spec, seed)
with Session(0) as s:
    s.set_scene(sc)
    hs = []
    for _ in range(n):
        r = s.reconstruct(cfg)
        h = hashlib.sha1(r["points"].tobytes() + r["background"].tobytes() + r["trace"].tobytes()).hexdigest()[:12]
        hs.append((h, r["iterations"], len(r["points"])))
    print(hs, flush=True)
