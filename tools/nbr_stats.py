"""Neighbour-scan statistics of a workload's cloud after a few PALM
iterations (GPU reconstruct, numpy/scipy here): points per coarse pixel, the
APSS window candidates per point (the kernel's disc-culled coarse rows) and
the ball members per point.  usage: python tools/nbr_stats.py [B|C|E] [iters]"""
import json
import sys
from pathlib import Path

import numpy as np
from scipy.spatial import cKDTree

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))
import workloads as W  # noqa: E402
from paper_1905_06700_b200.rt3d import Session  # noqa: E402
from scenegen.scene import simulate  # noqa: E402

key = sys.argv[1] if len(sys.argv) > 1 else "B"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 5
name, spec, seed, cfg = W.CONFIGS[key]()
cfg.max_iters = iters
sc = simulate(spec, seed)
with Session(0) as s:
    s.set_scene(sc)
    s.reconstruct_async(cfg)
    s.synchronize()
    pts, _ = s.state()
S = spec.superres
pf = spec.pixel_pitch_m  # the fine pitch (coarse = pitch x superres)
R = cfg.apss_radius
Wd = int(np.floor(R / pf)) + 1
fi = np.rint(pts["x"] / pf - 0.5).astype(np.int64)
fj = np.rint(pts["y"] / pf - 0.5).astype(np.int64)
rows, cols = spec.rows, spec.cols
cnt = np.bincount(pts["i"].astype(np.int64) * cols + pts["j"], minlength=rows * cols).reshape(rows, cols)
pre = np.concatenate([np.zeros((rows, 1), np.int64), np.cumsum(cnt, axis=1)], axis=1)
rng = np.random.default_rng(0)
qs = rng.choice(len(pts), size=min(len(pts), 20000), replace=False)
rw = R / pf
lim2 = rw * rw * (1 + 1e-9)
cand = np.zeros(len(qs), np.int64)
for n, q in enumerate(qs):
    a0, a1 = max(fi[q] - Wd, 0), min(fi[q] + Wd, rows * S - 1)
    tot = 0
    for ci in range(a0 // S, a1 // S + 1):
        rl, rh = ci * S, ci * S + S - 1
        dmin = rl - fi[q] if fi[q] < rl else (fi[q] - rh if fi[q] > rh else 0)
        rem = lim2 - dmin * dmin
        if rem < 0:
            continue
        wj = min(int(np.floor(np.sqrt(rem))), Wd)
        b0, b1 = max(fj[q] - wj, 0), min(fj[q] + wj, cols * S - 1)
        tot += pre[ci, b1 // S + 1] - pre[ci, b0 // S]
    cand[n] = tot
xyz = np.column_stack([pts["x"], pts["y"], pts["z"]])
tree = cKDTree(xyz)
mem = tree.query_ball_point(xyz[qs], R, return_length=True)
pp = np.bincount(cnt.ravel())
print(json.dumps({"config": key, "points": int(len(pts)), "W": Wd,
                  "points_per_pixel_hist": pp.tolist()[:12],
                  "cand_mean": float(cand.mean()), "cand_p90": float(np.percentile(cand, 90)),
                  "mem_mean": float(mem.mean()), "mem_p90": float(np.percentile(mem, 90)),
                  "mem_max": int(mem.max()), "frac_mem_gt_384": float((mem > 384).mean())}))

# candidates left after culling blocks of B consecutive points (aligned to
# each coarse pixel's first point) whose depth interval misses [z - R, z + R]
pix = pts["i"].astype(np.int64) * cols + pts["j"]
start = np.concatenate([[0], np.cumsum(cnt.ravel())])
z = pts["z"]
for B in (4, 8, 9):
    blk = (np.arange(len(pts)) - start[pix]) // B
    key = pix * 64 + blk
    uk, inv = np.unique(key, return_inverse=True)
    zmin = np.full(len(uk), np.inf)
    zmax = np.full(len(uk), -np.inf)
    np.minimum.at(zmin, inv, z)
    np.maximum.at(zmax, inv, z)
    kept = np.zeros(len(qs), np.int64)
    for n, q in enumerate(qs[:3000]):
        a0, a1 = max(fi[q] - Wd, 0), min(fi[q] + Wd, rows * S - 1)
        tot = 0
        for ci in range(a0 // S, a1 // S + 1):
            rl, rh = ci * S, ci * S + S - 1
            dmin = rl - fi[q] if fi[q] < rl else (fi[q] - rh if fi[q] > rh else 0)
            rem = lim2 - dmin * dmin
            if rem < 0:
                continue
            wj = min(int(np.floor(np.sqrt(rem))), Wd)
            b0, b1 = max(fj[q] - wj, 0), min(fj[q] + wj, cols * S - 1)
            lo, hi = start[ci * cols + b0 // S], start[ci * cols + b1 // S + 1]
            if hi > lo:
                ii = np.arange(lo, hi)
                ok = (zmin[inv[ii]] <= z[q] + R) & (zmax[inv[ii]] >= z[q] - R)
                tot += int(ok.sum())
        kept[n] = tot
    print(json.dumps({"block": B, "cand_kept_mean": float(kept[:3000].mean())}))
