"""GPU forward simulator: rt3d_simulate_cube samples
simulate_cube's photons (simulate.hpp:181-205) on the device.  Checked
against libscene's restatement, which is itself pinned bit for bit against
the reference's cubes (tests/test_scene.py).  The rates are bit-identical;
the samplers use libdevice exp/log/lgamma where the reference uses glibc's,
so the test allows a sample to differ only in a vanishing fraction of bins
(none were seen on the cases below)."""
import numpy as np
import pytest

from scenegen.scene import SceneSpec, SurfaceSpec, simulate
from test_scene import SPECS

MAX_DIFF_FRACTION = 1e-6   # of all (pixel, bin) samples


def _dense(offsets, events, npix, bins):
    z = np.zeros(npix * bins, np.uint64)
    pix = np.repeat(np.arange(npix), np.diff(offsets.astype(np.int64)))
    z[pix * bins + events["bin"].astype(np.int64)] = events["count"]
    return z


def _check(gpu, spec, seed):
    sc = simulate(spec, seed)
    gpu.set_scene(sc)
    n, sig, bgp = gpu.simulate_cube(sc.truth, sc.background_truth, seed)
    npix = spec.rows * spec.cols
    off, ev = gpu.cube_copy(npix, n)
    # CSR invariants (PhotonCube::validate, cube.hpp:84-112)
    assert off[0] == 0 and off[-1] == n and np.all(np.diff(off.astype(np.int64)) >= 0)
    assert np.all(ev["count"] >= 1) and np.all(ev["bin"] < spec.bins)
    if np.array_equal(off, sc.offsets) and np.array_equal(ev, sc.events):
        assert sig == sc.signal_photons and bgp == sc.background_photons
        return 0
    a = _dense(off, ev, npix, spec.bins)
    b = _dense(sc.offsets, sc.events, npix, spec.bins)
    diff = int(np.count_nonzero(a != b))
    assert diff <= MAX_DIFF_FRACTION * npix * spec.bins, diff
    return diff


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(SPECS))
def test_device_simulate_matches_restatement(gpu, name):
    spec, seed = SPECS[name]
    _check(gpu, spec, seed)


@pytest.mark.gpu
def test_device_simulate_dead_pixels_holes_checker(gpu):
    spec = SceneSpec(rows=20, cols=18, bins=400, bin_resolution_m=0.005, pixel_pitch_m=0.01,
                     target_ppp=5, target_sbr=4, dead_pixels=[(1, 2), (7, 7)],
                     surfaces=[SurfaceSpec(depth_m=1.2, holes=[(3, 3, 9, 9), (12, 0, 15, 4)]),
                               SurfaceSpec(kind="bump", depth_m=1.0, bump_amp=-0.1, bump_cx=0.1,
                                           bump_cy=0.09, bump_width=0.05, region=(2, 2, 17, 16),
                                           checker_contrast=0.3, checker_period=4)])
    _check(gpu, spec, 77)


@pytest.mark.gpu
def test_device_simulate_bright_pixels_take_ptrd(gpu):
    """target_ppp high enough that signal bins exceed lambda = 10 (PTRD branch,
    rng.hpp:63-96, with lgamma / log)."""
    spec = SceneSpec(rows=16, cols=16, bins=153, bin_resolution_m=0.0375, pixel_pitch_m=0.05,
                     target_ppp=900, target_sbr=1, superres=3,
                     surfaces=[SurfaceSpec(depth_m=1.5, region=(0, 0, 48, 20)),
                               SurfaceSpec(depth_m=3.0)])
    _check(gpu, spec, 1000)


@pytest.mark.gpu
def test_device_simulate_config_b_then_reconstruct(gpu):
    """BASELINE config B: the sampled cube is the session's cube, so a
    reconstruction runs on it directly and equals one on the host cube."""
    import bench
    spec, seed, cfg, _ = bench.config_b()
    _check(gpu, spec, seed)
    a = gpu.reconstruct(cfg)
    sc = simulate(spec, seed)
    gpu.set_scene(sc)
    b = gpu.reconstruct(cfg)
    assert np.array_equal(a["points"], b["points"])


@pytest.mark.gpu
def test_device_simulate_is_deterministic(gpu):
    spec, seed = SPECS["dense_12"]
    sc = simulate(spec, seed)
    gpu.set_scene(sc)
    n1, *_ = gpu.simulate_cube(sc.truth, sc.background_truth, seed)
    c1 = gpu.cube_copy(spec.rows * spec.cols, n1)
    n2, *_ = gpu.simulate_cube(sc.truth, sc.background_truth, seed)
    c2 = gpu.cube_copy(spec.rows * spec.cols, n2)
    assert np.array_equal(c1[0], c2[0]) and np.array_equal(c1[1], c2[1])
    n3, *_ = gpu.simulate_cube(sc.truth, sc.background_truth, seed + 1)
    c3 = gpu.cube_copy(spec.rows * spec.cols, n3)
    assert not (n3 == n1 and np.array_equal(c3[1], c1[1]))
