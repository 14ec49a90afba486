"""CPU: libscene.so (a restatement of simulate_cube, simulate.hpp:139-223)
reproduces the reference's cubes bit for bit (committed golden cubes made by
the reference; live against oracle/_ref when present)."""
import numpy as np
import pytest

import golden_io as G
import oracle_lib as O
from scenegen.scene import SceneSpec, SurfaceSpec, simulate

SPECS = {
    "small_s3": (SceneSpec(rows=16, cols=16, bins=300, bin_resolution_m=0.01, pixel_pitch_m=0.02,
                           target_ppp=6, target_sbr=10, surfaces=[SurfaceSpec(depth_m=1.5)]), 3),
    "two_surface_24": (SceneSpec(rows=24, cols=24, bins=750, bin_resolution_m=0.01,
                                 pixel_pitch_m=0.02, target_ppp=3, target_sbr=13,
                                 surfaces=[SurfaceSpec(depth_m=7.0),
                                           SurfaceSpec(depth_m=5.0, region=(6, 6, 18, 18))]), 1234),
    "superres_8": (SceneSpec(rows=8, cols=8, bins=200, superres=3, bin_resolution_m=0.01,
                             pixel_pitch_m=0.05, target_ppp=15, target_sbr=10,
                             surfaces=[SurfaceSpec(depth_m=1.0, slope_x=0.5)]), 11),
    "dense_12": (SceneSpec(rows=12, cols=12, bins=153, bin_resolution_m=0.0375,
                           pixel_pitch_m=0.05, target_ppp=60, target_sbr=1,
                           surfaces=[SurfaceSpec(depth_m=1.5, region=(0, 0, 12, 6)),
                                     SurfaceSpec(kind="bump", depth_m=3.0, bump_amp=-0.5,
                                                 bump_cx=0.3, bump_cy=0.3, bump_width=0.15),
                                     SurfaceSpec(depth_m=4.5)]), 5),
}


@pytest.mark.parametrize("name", sorted(SPECS))
def test_scene_matches_reference_cube(name):
    spec, seed = SPECS[name]
    got = simulate(spec, seed, threads=3)
    ref, _, _ = G.scene(name)
    assert np.array_equal(got.offsets, ref.offsets)
    assert np.array_equal(got.events, ref.events)
    assert np.array_equal(got.irf_samples, ref.irf_samples)
    assert got.irf_tau_min == ref.irf_tau_min and got.bin_width_s == ref.bin_width_s


def test_scene_thread_count_invariant():
    spec, seed = SPECS["dense_12"]
    a, b = simulate(spec, seed, threads=1), simulate(spec, seed, threads=7)
    assert np.array_equal(a.events, b.events) and np.array_equal(a.offsets, b.offsets)


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_scene_live_vs_reference_with_holes_and_dead_pixels():
    spec = SceneSpec(rows=20, cols=18, bins=400, bin_resolution_m=0.005, pixel_pitch_m=0.01,
                     target_ppp=5, target_sbr=4, dead_pixels=[(1, 2), (7, 7)],
                     surfaces=[SurfaceSpec(depth_m=1.2, holes=[(3, 3, 9, 9), (12, 0, 15, 4)]),
                               SurfaceSpec(kind="bump", depth_m=1.0, bump_amp=-0.1, bump_cx=0.1,
                                           bump_cy=0.09, bump_width=0.05, region=(2, 2, 17, 16),
                                           checker_contrast=0.3, checker_period=4)])
    text = """rows = 20
cols = 18
bins = 400
bin_resolution_m = 0.005
pixel_pitch_m = 0.01
target_ppp = 5
target_sbr = 4
dead_pixels = 1,2; 7,7
[surface]
depth_m = 1.2
holes = 3,3,9,9; 12,0,15,4
[surface]
type = bump
depth_m = 1.0
bump_amp = -0.1
bump_cx = 0.1
bump_cy = 0.09
bump_width = 0.05
region = 2,2,17,16
checker_contrast = 0.3
checker_period = 4
"""
    got = simulate(spec, 77)
    ref = O.ref_simulate(text, 77)
    assert np.array_equal(got.offsets, ref.offsets)
    assert np.array_equal(got.events, ref.events)
    assert np.array_equal(got.dead, ref.dead)
