import sys, ctypes as C, numpy as np
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import golden_io as G, bench
from paper_1905_06700_b200 import rt3d
from scenegen.scene import simulate
L = rt3d.lib()
L.rt3d_debug_clocks.argtypes = [C.c_void_p, C.POINTER(C.c_uint64)]
for name in ["small_s3", "B"]:
    if name == "B":
        spec, seed, cfg, _ = bench.config_b(); sc = simulate(spec, seed)
    else:
        sc, cfg, _ = G.scene(name)
    cfg.max_iters = 1
    with rt3d.Session(0) as s:
        s.set_scene(sc)
        s.reconstruct_async(cfg); s.synchronize()
        s.reconstruct_async(cfg); s.synchronize()
        buf = np.zeros(64, np.uint64)
        L.rt3d_debug_clocks(s.h, buf.ctypes.data_as(C.POINTER(C.c_uint64)))
        print(name, "stages: meta | copy-ev | points | sync | groups | sync")
        for kind in range(7):
            b = buf[kind*8: kind*8+7].astype(np.int64)
            if b[0]: print("  kind", kind, "deltas", np.diff(b))
