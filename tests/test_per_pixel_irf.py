"""Per-pixel IRFs (SensorModel::irf_per_pixel, sensor.hpp:160-164): every
pixel carries its own sampled Gaussian (sigma and sample spacing vary, so
the supports, the power-of-two and the true-division paths of Irf::value and
the global IRF table all get exercised).

CPU: the C oracle against the reference compiled unchanged (libref).
GPU: the CUDA path against both, at the north-star bars (init and the
likelihood sweeps bit-exact, reconstruct within tolerance, every PALM step
within tolerance of the reference's step).
"""
import numpy as np
import pytest

import golden_io as G
import oracle_lib as O
import parity as PY

needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref/libref.so not built")


def per_pixel_scene(name="two_surface_24"):
    sc, cfg, d = G.scene(name)
    irfs = []
    for p in range(sc.n_pixels):
        i, j = divmod(p, sc.n_cols)
        sigma = 1.0 + 0.25 * ((7 * i + 3 * j) % 5)
        dtau = 0.25 if (i + j) % 3 else 0.2   # 0.2: Irf::value's true division
        smp, tmin = O.irf_gaussian(sigma, 4.0, dtau)
        irfs.append((smp, tmin, dtau))
    sc.irf_per_pixel = irfs
    return sc, cfg


@needs_ref
def test_oracle_matches_reference_with_per_pixel_irfs():
    sc, cfg = per_pixel_scene()
    pts, bg = O.init_matched_filter(sc, cfg, "oracle")
    rp, rbg = O.init_matched_filter(sc, cfg, "ref")
    assert np.array_equal(pts, rp) and np.array_equal(bg, rbg)
    sc.with_state(pts, bg)
    a, b = O.grads(sc, "oracle"), O.grads(sc, "ref")
    for k in a:
        assert np.array_equal(a[k], b[k]), k
    assert O.nll(sc, "oracle") == O.nll(sc, "ref")


@pytest.mark.gpu
def test_gpu_init_and_sweeps_per_pixel_irfs(gpu):
    sc, cfg = per_pixel_scene()
    gpu.set_scene(sc)
    pts, bg = gpu.init_matched_filter(cfg)
    opts, obg = O.init_matched_filter(sc, cfg, "oracle")
    assert np.array_equal(pts, opts) and np.array_equal(bg, obg)
    sc.with_state(pts, bg)
    gpu.upload_state(sc.points, sc.background)
    ours, ref = gpu.grads(), O.grads(sc, "oracle")
    for k in ("gd", "gr", "gb", "cd", "cr", "cb", "oog"):
        assert np.array_equal(ours[k], ref[k]), k
    assert abs(gpu.nll() - O.nll(sc, "oracle")) <= 1e-13 * abs(O.nll(sc, "oracle"))


@pytest.mark.gpu
def test_gpu_reconstruct_per_pixel_irfs(gpu):
    sc, cfg = per_pixel_scene()
    d = PY.free_running(gpu, sc, cfg, "oracle")
    assert PY.within_tolerance(d) and d["backtracks_equal"] and d["flags_equal"], d


@pytest.mark.gpu
@needs_ref
def test_gpu_palm_steps_vs_reference_per_pixel_irfs(gpu):
    sc, cfg = per_pixel_scene()
    w = PY.stepwise(gpu, sc, cfg, "ref")
    assert w["same_cells"] and w["max_dt_bins"] <= PY.T_TOL_BINS, w
    assert w["max_rel_dr"] <= PY.R_TOL_REL and w["backtracks_equal"], w
