import os, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tools"))
import workloads as W
from paper_1905_06700_b200.rt3d import Session
from scenegen.scene import simulate
name, spec, seed, cfg = W.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "D"]()
cfg.max_iters = 4
with Session(0) as s:
    s.set_scene(simulate(spec, seed))
    s.time_kernels(True)
    try:
        s.reconstruct_async(cfg)
        s.synchronize()
        print("ok", s.kernel_times())
    except Exception as e:
        print("ERR", e)
