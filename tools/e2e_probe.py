"""Where the e2e step's time goes (config B, batches of 16, bench.py's e2e
loop): wall time of the 16 rt3d_set_cube calls, of rt3d_reconstruct_batch up
to completion, and of the 16 rt3d_state_size + rt3d_state_copy calls."""
import copy
import ctypes as C
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import config_b  # noqa: E402
from paper_1905_06700_b200 import rt3d as R  # noqa: E402
from paper_1905_06700_b200.abi import POINT_DTYPE  # noqa: E402
from paper_1905_06700_b200.rt3d import Session  # noqa: E402
from scenegen.scene import simulate  # noqa: E402

NB = 16
spec, seed, cfg, _ = config_b()
cubes = [simulate(spec, seed + k) for k in range(NB)]
ss = [Session(0) for _ in range(NB)]
pinned = []
for s, c in zip(ss, cubes):
    s.set_scene(c)
    cp = copy.copy(c)
    off = torch.empty(len(c.offsets), dtype=torch.int64, pin_memory=True).numpy().view(np.uint64)
    ev = torch.empty(len(c.events) * 2, dtype=torch.int32, pin_memory=True).numpy().view(c.events.dtype)
    off[:] = c.offsets
    ev[:] = c.events
    cp.offsets, cp.events = off, ev
    pinned.append(cp)
P_cap = cfg.init_max_returns * spec.superres * spec.superres * cubes[0].n_pixels
outs = [(torch.empty(P_cap * 64, dtype=torch.uint8, pin_memory=True).numpy().view(POINT_DTYPE),
         torch.empty(cubes[0].n_pixels, dtype=torch.float64, pin_memory=True).numpy())
        for _ in range(NB)]
acc = {"set_cube": 0.0, "batch": 0.0, "download": 0.0}
steps = 8
for k in range(steps + 2):
    t0 = time.perf_counter()
    for s, c in zip(ss, pinned):
        s.set_cube(c)
    t1 = time.perf_counter()
    Session.reconstruct_batch_async(ss, cfg)
    ss[0].synchronize()
    t2 = time.perf_counter()
    for s, (op, ob) in zip(ss, outs):
        n = R._u64()
        R._check(R.lib().rt3d_state_size(s.h, C.byref(n)))
        R._check(R.lib().rt3d_state_copy(s.h, R.ptr(op, R.Point), R.ptr(ob, R._dbl)))
    t3 = time.perf_counter()
    if k >= 2:
        acc["set_cube"] += (t1 - t0) / steps * 1e3
        acc["batch"] += (t2 - t1) / steps * 1e3
        acc["download"] += (t3 - t2) / steps * 1e3
print(json.dumps({"ms_per_step": acc}), flush=True)
