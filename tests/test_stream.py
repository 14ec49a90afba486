"""GPU: the streaming API (rt3d_frame_submit / rt3d_frame_collect) on a
stream of different cubes — different seeds, so different event counts —
gives, frame by frame, what reconstruct gives on that cube; plus the
collect / validation error paths (include/rt3d.h)."""
import numpy as np
import pytest

from paper_1905_06700_b200.abi import Config
from paper_1905_06700_b200.rt3d import Rt3dError, Session
from scenegen.scene import SceneSpec, SurfaceSpec, simulate

pytestmark = pytest.mark.gpu

SPEC = SceneSpec(rows=20, cols=20, bins=400, bin_resolution_m=0.01, pixel_pitch_m=0.02,
                 target_ppp=8.0, target_sbr=4.0,
                 surfaces=[SurfaceSpec(depth_m=2.0),
                           SurfaceSpec(depth_m=1.5, region=(5, 5, 14, 14))])
CFG = Config(max_iters=6, stop_tol=0.0, apss_radius=0.1, knn_k=5, r_min=0.2,
             init_max_returns=2, init_min_separation=6)


def test_stream_of_different_cubes_matches_reconstruct(gpu):
    cubes = [simulate(SPEC, seed) for seed in (11, 12, 13, 14, 15)]
    assert len({len(c.events) for c in cubes}) > 1          # event counts differ
    refs = []
    for c in cubes:
        gpu.set_scene(c)
        refs.append(gpu.reconstruct(CFG))
    with Session(0) as s:
        s.set_scene(cubes[0])
        pend = []
        got = []
        for k, c in enumerate(cubes + cubes):                # twice: cached graphs replay
            if len(pend) == 2:
                got.append(s.frame_collect(pend.pop(0)))
            pend.append(s.frame_submit(c, CFG))
        got += [s.frame_collect(t) for t in pend]
    for k, (pts, bg, rep) in enumerate(got):
        ref = refs[k % len(cubes)]
        assert np.array_equal(pts, ref["points"]), k
        assert np.array_equal(bg, ref["background"]), k
        assert rep["final_nll"] == ref["trace"][-1], k


def test_stream_of_different_cubes_replays_one_graph(gpu):
    """Frames of a stream differ in their cubes, not in their launch
    parameters: one captured graph serves them all (a key holding
    per-cube sizes would re-capture every frame)."""
    cubes = [simulate(SPEC, seed) for seed in (31, 32, 33, 34, 35, 36)]
    assert len({len(c.events) for c in cubes}) > 1

    def stream(s):
        pend = [s.frame_submit(c, CFG) for c in cubes[:2]]
        for c in cubes[2:]:
            s.frame_collect(pend.pop(0))
            pend.append(s.frame_submit(c, CFG))
        for t in pend:
            s.frame_collect(t)

    with Session(0) as s:
        s.set_scene(cubes[0])
        stream(s)                       # buffers grow to the stream's sizes
        c0, n0 = s.graph_counts()
        assert c0 <= 4                  # (a graph per in-flight slot, and growth)
        stream(s)
        c1, n1 = s.graph_counts()
    assert n1 - n0 == len(cubes)
    assert c1 == c0                     # every frame of the second pass replays


def test_collect_with_too_small_buffer_keeps_the_frame(gpu):
    c = simulate(SPEC, 21)
    gpu.set_scene(c)
    ref = gpu.reconstruct(CFG)
    assert len(ref["points"]) > 1
    t = gpu.frame_submit(c, CFG)
    small = np.zeros(1, ref["points"].dtype)
    with pytest.raises(Rt3dError) as e:
        gpu.frame_collect(t, small)
    assert e.value.status == 3                                # OUT_OF_RANGE
    pts, bg, _ = gpu.frame_collect(t)                         # still collectable
    assert np.array_equal(pts, ref["points"])
    assert np.array_equal(bg, ref["background"])


def test_fft_background_needs_a_2x2_image(gpu):
    """reconstruct -> palm_step -> fft_background_denoise throws
    invalid_argument on a 1xN image (denoise.hpp:269-270)."""
    spec = SceneSpec(rows=1, cols=8, bins=200, target_ppp=5.0, target_sbr=5.0,
                     surfaces=[SurfaceSpec(depth_m=1.0)])
    c = simulate(spec, 3)
    cfg = Config(max_iters=2, stop_tol=0.0, apss_radius=0.1, background_mode=1, fft_cutoff=0.5)
    gpu.set_scene(c)
    with pytest.raises(Rt3dError) as e:
        gpu.reconstruct(cfg)
    assert e.value.status == 1 and "2x2" in str(e.value)
    with pytest.raises(Rt3dError) as e:
        gpu.frame_submit(c, cfg)
    assert e.value.status == 1
