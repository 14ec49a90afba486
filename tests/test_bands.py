"""GPU: one frame split into row bands (rt3d_reconstruct_bands, SURVEY.md
§8e config E's decomposition) equals the single-band reconstruction bit for
bit: the bands own subtrees of pairwise_sum's pixel tree, read their
neighbours' halo rows through halo_kernel before APSS and kNN, and share one
grid barrier, one prune / spawn scan and one block-node tree.  Each band is
its own session with its own buffers, so a stale or missing halo row, a
wrong scan base or a wrong tree combination shows up as a difference."""
import numpy as np
import pytest

import workloads as W
from paper_1905_06700_b200.abi import Config
from paper_1905_06700_b200.rt3d import Rt3dError, Session
from scenegen.scene import SceneSpec, simulate

pytestmark = pytest.mark.gpu


def _same(a, b):
    assert len(a["points"]) == len(b["points"])
    assert np.array_equal(a["points"], b["points"])
    assert np.array_equal(a["background"], b["background"])
    assert np.array_equal(a["trace"], b["trace"])
    assert np.array_equal(a["steps"], b["steps"])
    assert a["iterations"] == b["iterations"] and a["points"].size == b["points"].size


def _bands(sc, cfg, n):
    ss = [Session(0) for _ in range(n)]
    try:
        for s in ss:
            s.set_scene(sc)
        return Session.reconstruct_bands(ss, cfg)
    finally:
        for s in ss:
            s.close()


def _scene(rows, bins, seed, ppp=30.0):
    spec = SceneSpec(rows=rows, cols=rows, bins=bins, bin_resolution_m=0.01, pixel_pitch_m=0.02,
                     irf_sigma_bins=1.5, target_ppp=ppp, target_sbr=1.0,
                     surfaces=W._camouflage(rows, max(1, rows // 256)))
    return simulate(spec, seed)


@pytest.mark.parametrize("n", [1, 2, 4, 8, 16])
def test_bands_equal_single_frame_large_array(gpu, n):
    """256x256x2048 (config D, thread-per-pixel sweeps)."""
    name, spec, seed, cfg = W.config_d()
    cfg.max_iters = 4
    sc = simulate(spec, seed)
    gpu.set_scene(sc)
    ref = gpu.reconstruct(cfg)
    _same(_bands(sc, cfg, n), ref)


@pytest.mark.parametrize("n", [2, 4])
def test_bands_equal_single_frame_lane_groups(gpu, n):
    """128x128 (warp-per-pixel sweeps), several prune steps."""
    sc = _scene(128, 1400, 77, ppp=20.0)
    cfg = W.acceptance_cfg(max_iters=6)
    gpu.set_scene(sc)
    ref = gpu.reconstruct(cfg)
    assert ref["steps"]["points_after"][-1] < ref["steps"]["points_before"][0]  # prune ran
    _same(_bands(sc, cfg, n), ref)


def test_band_errors(gpu):
    name, spec, seed, cfg = W.config_b()     # 141x141: the halves are not whole rows
    sc = simulate(spec, seed)
    with pytest.raises(Rt3dError) as e:
        _bands(sc, cfg, 2)
    assert e.value.status == 6
    sc = _scene(128, 1400, 3)
    cfg = W.acceptance_cfg(max_iters=2, background_mode=1)
    with pytest.raises(Rt3dError) as e:
        _bands(sc, cfg, 2)
    assert e.value.status == 6
    with pytest.raises(Rt3dError) as e:
        _bands(sc, W.acceptance_cfg(max_iters=2), 3)
    assert e.value.status == 1
