"""Time the device sampler (rt3d_simulate_cube) against libscene's threaded
host restatement of simulate_cube on BASELINE configs B and D-like.  Wall
clock around each call (the ABI call synchronises); the device figure includes
the host bucket sort and the truth/background upload."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_1905_06700_b200.rt3d import Session  # noqa: E402
from scenegen.scene import SceneSpec, SurfaceSpec, simulate  # noqa: E402


def config_d():
    spec = SceneSpec(rows=256, cols=256, bins=2048, bin_resolution_m=0.01, pixel_pitch_m=0.02,
                     target_ppp=30, target_sbr=1,
                     surfaces=[SurfaceSpec(depth_m=5.0, holes=[(a, b, a + 8, b + 8)
                                                             for a in range(0, 256, 16)
                                                             for b in range(0, 256, 16)]),
                               SurfaceSpec(kind="bump", depth_m=8.0, bump_amp=-0.5, bump_cx=2.56,
                                           bump_cy=2.56, bump_width=1.0),
                               SurfaceSpec(depth_m=12.0)])
    return spec, 256


out = {}
s = Session(0)
for name, (spec, seed) in {"B": bench.config_b()[:2], "D": config_d()}.items():
    t0 = time.perf_counter()
    sc = simulate(spec, seed)
    cpu = time.perf_counter() - t0
    s.set_scene(sc)
    s.simulate_cube(sc.truth, sc.background_truth, seed)  # warm-up
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        n, sig, bgp = s.simulate_cube(sc.truth, sc.background_truth, seed)
        ts.append(time.perf_counter() - t0)
    off, ev = s.cube_copy(spec.rows * spec.cols, n)
    same = bool(np.array_equal(off, sc.offsets) and np.array_equal(ev, sc.events))
    out[name] = {"pixels": spec.rows * spec.cols, "bins": spec.bins, "events": int(n),
                 "samples": 2 * spec.rows * spec.cols * spec.bins,
                 "cpu_s_all_threads": cpu, "cpu_threads": os.cpu_count(),
                 "gpu_s_median": float(np.median(ts)), "identical_to_host": same}
print(json.dumps(out))
