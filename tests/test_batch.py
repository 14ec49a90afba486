"""GPU: batched frames (rt3d_reconstruct_batch, a frame axis in every
kernel's grid) give, session by session, exactly what rt3d_reconstruct gives
on that session's cube: clouds, backgrounds, nll traces and step
diagnostics bit for bit, for batches of 1..32 frames of different cubes (single
frames and small batches take other kernel variants than large batches: the
split fit, two depth candidates per sweep, lane-group sweeps)."""
import numpy as np
import pytest

import workloads as W
from paper_1905_06700_b200.abi import Config
from paper_1905_06700_b200.rt3d import Rt3dError, Session
from scenegen.scene import SceneSpec, SurfaceSpec, simulate

pytestmark = pytest.mark.gpu

SPEC = SceneSpec(rows=24, cols=24, bins=500, bin_resolution_m=0.01, pixel_pitch_m=0.02,
                 target_ppp=6.0, target_sbr=5.0,
                 surfaces=[SurfaceSpec(depth_m=3.0),
                           SurfaceSpec(depth_m=2.0, region=(6, 6, 18, 18))])
CFG = Config(max_iters=6, stop_tol=0.0, apss_radius=0.12, knn_k=7, r_min=0.2,
             init_max_returns=2, init_min_separation=6)


def _same(a, b):
    assert np.array_equal(a["points"], b["points"])
    assert np.array_equal(a["background"], b["background"])
    assert np.array_equal(a["trace"], b["trace"])
    assert np.array_equal(a["steps"], b["steps"])
    assert a["iterations"] == b["iterations"]


def _batch(cubes, cfg):
    ss = [Session(0) for _ in cubes]
    try:
        for s, c in zip(ss, cubes):
            s.set_scene(c)
        Session.reconstruct_batch_async(ss, cfg)
        out = []
        for s in ss:
            r = s.report()
            r["points"], r["background"] = s.state()
            out.append(r)
        return out
    finally:
        for s in ss:
            s.close()


@pytest.mark.parametrize("n", [1, 2, 3, 8, 16, 32])
def test_batch_matches_single_frames(gpu, n):
    cubes = [simulate(SPEC, 40 + k) for k in range(n)]
    singles = []
    for c in cubes:
        gpu.set_scene(c)
        singles.append(gpu.reconstruct(CFG))
    for a, b in zip(_batch(cubes, CFG), singles):
        _same(a, b)


@pytest.mark.parametrize("key,n", [("B", 2), ("C", 4)])
def test_batch_of_benchmark_frames(gpu, key, n):
    name, spec, seed, cfg = W.CONFIGS[key]()
    cfg.max_iters = 5
    if key == "C":
        cubes = [simulate(W.config_c(f)[1], 1000 + f) for f in range(n)]
    else:
        cubes = [simulate(spec, seed)] * n
    singles = []
    for c in cubes:
        gpu.set_scene(c)
        singles.append(gpu.reconstruct(cfg))
    for a, b in zip(_batch(cubes, cfg), singles):
        _same(a, b)


def test_batch_errors(gpu):
    c = simulate(SPEC, 1)
    s1, s2 = Session(0), Session(0)
    try:
        s1.set_scene(c)
        s2.set_scene(c)
        with pytest.raises(Rt3dError) as e:
            Session.reconstruct_batch_async([s1, s1], CFG)
        assert e.value.status == 1
        # a dense and a sparse cube need different sweep layouts
        dense = simulate(SceneSpec(rows=24, cols=24, bins=500, target_ppp=80.0, target_sbr=0.5,
                                   surfaces=[SurfaceSpec(depth_m=3.0)]), 2)
        s2.set_scene(dense)
        with pytest.raises(Rt3dError) as e:
            Session.reconstruct_batch_async([s1, s2], CFG)
        assert e.value.status == 6
    finally:
        s1.close()
        s2.close()


def test_alternating_groups_pipeline(gpu):
    """bench.py's e2e pipeline: two groups of sessions alternate batches,
    each batch queued behind the other group's with rt3d_session_after, the
    next group's uploads issued before this group's downloads; every frame is
    what rt3d_reconstruct gives on its cube."""
    n, steps = 4, 4
    cubes = [simulate(SPEC, 70 + k) for k in range(n * steps)]
    singles = []
    for c in cubes:
        gpu.set_scene(c)
        singles.append(gpu.reconstruct(CFG))
    groups = [[Session(0) for _ in range(n)] for _ in range(2)]
    try:
        for g in groups:
            for s in g:
                s.set_scene(cubes[0])

        def launch(k):
            g = groups[k % 2]
            for s, c in zip(g, cubes[k * n:(k + 1) * n]):
                s.set_cube(c)
            g[0].after(groups[(k + 1) % 2][0])
            Session.reconstruct_batch_async(g, CFG)

        launch(0)
        for k in range(steps):
            if k + 1 < steps:
                launch(k + 1)
            for j, s in enumerate(groups[k % 2]):
                r = s.report()
                r["points"], r["background"] = s.state()
                _same(r, singles[k * n + j])
    finally:
        for g in groups:
            for s in g:
                s.close()
