"""One config-E frame (1024x1024x2048) for ncu: `ncu -k regex:stage_kernel
-s S -c C python tools/profile_e.py [iters]` (the warm-up frame is skipped
by -s).  Without ncu it prints the per-class kernel times."""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))
import workloads as W  # noqa: E402
from paper_1905_06700_b200.rt3d import Session  # noqa: E402
from scenegen.scene import simulate  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 2
name, spec, seed, cfg = W.config_e()
cfg.max_iters = iters
sc = simulate(spec, seed)
with Session(0) as s:
    s.set_scene(sc)
    s.time_kernels(True)
    s.reconstruct_async(cfg)
    kt = s.kernel_times()
    print(json.dumps({"events": int(len(sc.events)), "iters": iters,
                      "kernel_ms": {k: v for k, v in kt.items() if v[1]}}), flush=True)
