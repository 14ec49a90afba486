"""Frames/s with G concurrent batch groups (each its own sessions / stream,
cooperative grids sized for G groups with rt3d_session_set_sharing) of n
frames each, config B (or C): CUDA events on a side stream bracket K rounds
of all groups."""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_1905_06700_b200.rt3d import Session  # noqa: E402
from scenegen.scene import simulate  # noqa: E402

key = sys.argv[1] if len(sys.argv) > 1 else "B"
name, spec, seed, cfg = W.CONFIGS[key]()
cubes = [simulate(spec, seed + k) for k in range(16)] if key != "C" else \
    [simulate(W.config_c(f)[1], 1000 + f) for f in range(16)]
for G, n in ((1, 8), (2, 4), (2, 8)):
    groups = [[Session(0) for _ in range(n)] for _ in range(G)]
    try:
        for g, ss in enumerate(groups):
            for k, s in enumerate(ss):
                s.set_scene(cubes[(g * n + k) % len(cubes)])
                s.set_sharing(G)
        def round_():
            for ss in groups:
                Session.reconstruct_batch_async(ss, cfg)
        for _ in range(3):
            round_()
        torch.cuda.synchronize()
        K = 8
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        import time
        t0 = time.perf_counter()
        for _ in range(K):
            round_()
        for ss in groups:
            ss[0].synchronize()
        dt = time.perf_counter() - t0
        print(json.dumps({"config": key, "groups": G, "batch": n, "frames_per_s": K * G * n / dt}),
              flush=True)
    except Exception as e:  # noqa: BLE001
        print(json.dumps({"config": key, "groups": G, "batch": n, "error": str(e)}), flush=True)
    finally:
        for ss in groups:
            for s in ss:
                s.close()
