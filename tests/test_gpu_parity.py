"""GPU parity: the CUDA path (through the C ABI, librt3d.so) against the C
oracle on the same inputs.  Inputs are the reference's own generators'
outputs committed under tests/golden/ (random_instance, simulate_cube).

Bars (BASELINE.json north_star):
  - matched-filter peak lags / init points: bit-exact;
  - likelihood sweeps (gradients, curvatures): bit-exact (no FMA, IEEE
    division; -fmad=false on both sides).  The nll differs only through
    log(): libdevice vs glibc, <= 1 ulp per term -> relative 1e-13;
  - reconstruct: per-point depth within 1e-3 bins, intensity within 1e-4
    relative, surviving point count within 0.1% (north_star tolerances);
    in practice the trajectories are identical.
"""
import numpy as np
import pytest

import golden_io as G
import oracle_lib as O

pytestmark = pytest.mark.gpu

NLL_REL = 1e-13


def _close_nll(a, b, rel=NLL_REL):
    if np.isinf(a) or np.isinf(b):
        return a == b
    return abs(a - b) <= rel * max(1.0, abs(b))


@pytest.mark.parametrize("seed", G.random_seeds())
def test_likelihood_sweeps_random_instances(gpu, seed):
    sc, _ = G.random_instance(seed)
    gpu.set_scene(sc)
    gpu.upload_state(sc.points, sc.background)
    ours = gpu.grads()
    ref = O.grads(sc, "oracle")
    for k in ("gd", "gr", "gb", "cd", "cr", "cb", "oog"):
        assert np.array_equal(ours[k], ref[k]), (k, np.max(np.abs(ours[k] - ref[k])))
    assert _close_nll(gpu.nll(), O.nll(sc, "oracle"))


@pytest.mark.parametrize("name", G.SCENE_NAMES)
def test_init_bit_exact(gpu, name):
    sc, cfg, d = G.scene(name)
    gpu.set_scene(sc)
    pts, bg = gpu.init_matched_filter(cfg)
    opts, obg = O.init_matched_filter(sc, cfg, "oracle")
    assert np.array_equal(pts, opts)
    assert np.array_equal(bg, obg)
    # and against the reference's own output
    assert np.array_equal(pts, d["init_points"])


@pytest.mark.parametrize("name", G.SCENE_NAMES)
def test_nll_and_grads_after_init(gpu, name):
    sc, cfg, d = G.scene(name)
    sc.with_state(d["init_points"], d["init_background"])
    gpu.set_scene(sc)
    gpu.upload_state(sc.points, sc.background)
    ours = gpu.grads()
    ref = O.grads(sc, "oracle")
    for k in ("gd", "gr", "gb", "cd", "cr", "cb", "oog"):
        assert np.array_equal(ours[k], ref[k]), k
    assert _close_nll(gpu.nll(), O.nll(sc, "oracle"))


def test_matched_filter_peaks(gpu):
    pk = G.peaks()
    irf, tmin = pk["irf"], float(pk["tau_min"])
    from paper_1905_06700_b200.abi import EVENT_DTYPE
    for key in pk:
        if not key.endswith("_events"):
            continue
        case = key[: -len("_events")]
        name, k, thr, sep = case.split("_")
        ev = np.ascontiguousarray(pk[key], np.uint32).view(EVENT_DTYPE).reshape(-1)
        got = gpu.matched_filter_peaks(ev, irf, tmin, 0.25, 200, int(k), float(thr), int(sep))
        assert np.array_equal(got, pk[case]), case


@pytest.mark.parametrize("name", G.SCENE_NAMES)
def test_palm_step_matches_oracle(gpu, name):
    sc, cfg, d = G.scene(name)
    sc.with_state(d["init_points"], d["init_background"])
    gpu.set_scene(sc)
    gpu.upload_state(sc.points, sc.background)
    pts, bg, diag = gpu.palm_step(cfg)
    opts, obg, odiag = O.palm_step(sc, cfg, "oracle")
    assert len(pts) == len(opts)
    assert np.max(np.abs(pts["t"] - opts["t"]), initial=0) <= 1e-9
    np.testing.assert_allclose(pts["intensity"], opts["intensity"], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(bg, obg, rtol=1e-9, atol=1e-15)
    assert np.array_equal(pts["flags"], opts["flags"])
    for f in ("nll_before", "nll_after"):
        assert _close_nll(getattr(diag, f), getattr(odiag, f), 1e-10)
    assert diag.depth.backtracks == odiag.depth.backtracks
    assert diag.intensity.backtracks == odiag.intensity.backtracks
    assert diag.background.backtracks == odiag.background.backtracks


def _assert_recon_parity(rep, ref, label):
    a, b = rep["points"], ref["points"]
    n, m = len(a), len(b)
    assert abs(n - m) <= max(0.001 * m, 0), (label, n, m)
    if n == m and n:
        assert np.array_equal(a["i"], b["i"]) and np.array_equal(a["fi"], b["fi"])
        dt = np.max(np.abs(a["t"] - b["t"]))
        dr = np.max(np.abs(a["intensity"] - b["intensity"]) /
                    np.maximum(np.abs(b["intensity"]), 1e-300))
        assert dt <= 1e-3, (label, dt)
        assert dr <= 1e-4, (label, dr)
    np.testing.assert_allclose(rep["trace"], ref["trace"], rtol=1e-9)


@pytest.mark.parametrize("name", G.SCENE_NAMES)
def test_reconstruct_matches_oracle(gpu, name):
    sc, cfg, d = G.scene(name)
    gpu.set_scene(sc)
    rep = gpu.reconstruct(cfg)
    ref = O.reconstruct(sc, cfg, "oracle")
    assert rep["iterations"] == ref["iterations"]
    _assert_recon_parity(rep, ref, name)
    # and against the reference's own run (Eigen stand-in differs at 1e-11)
    _assert_recon_parity(rep, {"points": d["rec_points"], "trace": d["rec_trace"]}, name + "/ref")


def test_reconstruct_deterministic(gpu):
    sc, cfg, _ = G.scene("two_surface_24")
    gpu.set_scene(sc)
    a = gpu.reconstruct(cfg)
    b = gpu.reconstruct(cfg)
    assert np.array_equal(a["points"], b["points"])
    assert np.array_equal(a["background"], b["background"])
    assert np.array_equal(a["trace"], b["trace"])


@pytest.mark.parametrize("name", G.SCENE_NAMES)
def test_baseline_xcorr(gpu, name):
    sc, cfg, d = G.scene(name)
    gpu.set_scene(sc)
    got = gpu.baseline_xcorr()
    assert np.array_equal(got, O.baseline_xcorr(sc, "oracle"))
    assert np.array_equal(got, d["baseline_points"])


def test_general_cloud_denoisers(gpu):
    d = G.denoise()
    for cloud, r in (("sphere", 0.45), ("noisy", 0.2)):
        got = gpu.apss_project(d[cloud], r)
        exp = O.apss_project(d[cloud], r, impl="oracle")
        assert np.array_equal(got["flags"], exp["flags"])
        for k in "xyz":
            assert np.max(np.abs(got[k] - exp[k])) <= 1e-12, (cloud, k)
    for k in (1, 6):
        got = gpu.knn_filter(d["noisy"], k, 0.25)
        assert np.array_equal(got, O.knn_filter(d["noisy"], k, 0.25, impl="oracle"))
        assert np.array_equal(got, d[f"noisy_knn{k}"])
    pr = gpu.prune(d["noisy"], 2.0)
    exp = d["noisy"][d["noisy"]["intensity"] >= 2.0]
    assert np.array_equal(pr, exp)


def test_fft_lowpass(gpu):
    d = G.denoise()
    np.testing.assert_allclose(gpu.fft_lowpass(d["img"], 0.4), d["img_fft04"], atol=1e-12)
    np.testing.assert_allclose(gpu.fft_lowpass(d["img"], 0.4, clamp=True), d["img_fft04_clamp"],
                               atol=1e-12)
    img = d["img"]
    np.testing.assert_allclose(gpu.fft_lowpass(img, 1.0), img, atol=1e-12)


def _recon_with_env(gpu, sc, cfg, env):
    import os
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        gpu.set_scene(sc)
        return gpu.reconstruct(cfg)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


@pytest.mark.parametrize("name", G.SCENE_NAMES + ["config_b"])
def test_knn_window_pruning_is_exact(gpu, name):
    """The kNN kernel's window pruning (knn_warps) selects exactly the
    neighbours of the full-ball scan: bit-identical reconstructions,
    including the full-size bench frame."""
    if name == "config_b":
        import sys
        from pathlib import Path
        sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
        import bench
        from scenegen.scene import simulate
        spec, seed, cfg, _ = bench.config_b()
        cfg.max_iters = 4
        sc = simulate(spec, seed)
    else:
        sc, cfg, _ = G.scene(name)
    a = _recon_with_env(gpu, sc, cfg, {})
    b = _recon_with_env(gpu, sc, cfg, {"RT3D_KNN_NO_PRUNE": "1"})
    assert np.array_equal(a["points"], b["points"])
    assert np.array_equal(a["background"], b["background"])
    assert np.array_equal(a["trace"], b["trace"])


@pytest.mark.parametrize("gsz", ["3", "4", "32"])
@pytest.mark.parametrize("name", G.SCENE_NAMES)
def test_lane_group_configs_agree(gpu, name, gsz):
    """Every lane-group configuration of the likelihood sweeps (3 or 4 lanes
    per pixel, or a warp per pixel) gives the same bits."""
    sc, cfg, _ = G.scene(name)
    a = _recon_with_env(gpu, sc, cfg, {})
    b = _recon_with_env(gpu, sc, cfg, {"RT3D_GSZ": gsz})
    assert np.array_equal(a["points"], b["points"])
    assert np.array_equal(a["background"], b["background"])
    assert np.array_equal(a["trace"], b["trace"])


@pytest.mark.parametrize("name", G.SCENE_NAMES)
def test_blocktree_and_barrier_tree_reductions_agree(gpu, name):
    """The block-node reduction with replicated controllers (default) and
    the barrier-separated last-block reduction give the same bits."""
    sc, cfg, _ = G.scene(name)
    a = _recon_with_env(gpu, sc, cfg, {})
    b = _recon_with_env(gpu, sc, cfg, {"RT3D_TREE_OLD": "1"})
    assert np.array_equal(a["points"], b["points"])
    assert np.array_equal(a["background"], b["background"])
    assert np.array_equal(a["trace"], b["trace"])


def test_pipelined_frames_match_reconstruct(gpu):
    """rt3d_frame_submit / rt3d_frame_collect with two frames in flight give
    the same clouds, backgrounds and reports as reconstruct, frame by frame."""
    scenes = [G.scene(n) for n in ("small_s3", "two_surface_24")]
    # same sensor per session: use one scene's sensor with two seeds' cubes
    sc, cfg, _ = scenes[1]
    gpu.set_scene(sc)
    ref = gpu.reconstruct(cfg)
    tickets = [gpu.frame_submit(sc, cfg) for _ in range(2)]
    for t in tickets:
        pts, bg, rep = gpu.frame_collect(t)
        assert np.array_equal(pts, ref["points"])
        assert np.array_equal(bg, ref["background"])
        assert rep["iterations"] == ref["iterations"]
        assert rep["final_nll"] == ref["trace"][-1]
    with pytest.raises(Exception):
        gpu.frame_collect(tickets[0])      # already collected
    t3 = gpu.frame_submit(sc, cfg)
    t4 = gpu.frame_submit(sc, cfg)
    with pytest.raises(Exception):
        gpu.frame_submit(sc, cfg)          # a third frame in flight
    for t in (t3, t4):
        pts, bg, _ = gpu.frame_collect(t)
        assert np.array_equal(pts, ref["points"])
    # the resident-state API still works after pipelined frames
    again = gpu.reconstruct(cfg)
    assert np.array_equal(again["points"], ref["points"])


@pytest.mark.parametrize("name", G.SCENE_NAMES + ["config_b"])
def test_two_candidate_sweeps_agree(gpu, name):
    """Depth / intensity candidate sweeps that evaluate alpha and alpha*beta
    together (default) take exactly the decisions of one-candidate sweeps."""
    if name == "config_b":
        import sys
        from pathlib import Path
        sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
        import bench
        from scenegen.scene import simulate
        spec, seed, cfg, _ = bench.config_b()
        cfg.max_iters = 6
        sc = simulate(spec, seed)
    else:
        sc, cfg, _ = G.scene(name)
    a = _recon_with_env(gpu, sc, cfg, {})
    b = _recon_with_env(gpu, sc, cfg, {"RT3D_ONE_CAND": "1"})
    assert np.array_equal(a["points"], b["points"])
    assert np.array_equal(a["background"], b["background"])
    assert np.array_equal(a["trace"], b["trace"])
    assert np.array_equal(a["steps"], b["steps"])


def test_large_array_one_candidate_default_agrees(gpu):
    """Frames of 2^20+ events default to one-candidate intensity sweeps
    (rt3d.cu build_frame); on config D they take exactly the decisions of
    forced two-candidate sweeps (both blocks)."""
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tools"))
    import bench_configs
    from scenegen.scene import simulate
    _, spec, seed, cfg = bench_configs.config_d()
    cfg.max_iters = 3
    sc = simulate(spec, seed)
    assert len(sc.events) >= (1 << 20)       # takes the large-array default
    a = _recon_with_env(gpu, sc, cfg, {})
    b = _recon_with_env(gpu, sc, cfg, {"RT3D_TWO_CAND": "3"})
    assert np.array_equal(a["points"], b["points"])
    assert np.array_equal(a["background"], b["background"])
    assert np.array_equal(a["trace"], b["trace"])
    assert np.array_equal(a["steps"], b["steps"])


def test_concurrent_sessions_match_sequential(gpu):
    """Two sessions sized to share the device (rt3d_session_set_sharing)
    reconstructing alternate frames concurrently give the sequential results."""
    from paper_1905_06700_b200.rt3d import Session
    sc, cfg, _ = G.scene("two_surface_24")
    gpu.set_scene(sc)
    ref = gpu.reconstruct(cfg)
    ss = [Session(0), Session(0)]
    try:
        for s in ss:
            s.set_scene(sc)
            s.set_sharing(2)
        pend = []
        for k in range(8):
            s = ss[k % 2]
            pend.append((s, s.frame_submit(sc, cfg)))
            if len(pend) == 4:
                ps, pt = pend.pop(0)
                pts, bg, _ = ps.frame_collect(pt)
                assert np.array_equal(pts, ref["points"])
                assert np.array_equal(bg, ref["background"])
        for ps, pt in pend:
            pts, bg, _ = ps.frame_collect(pt)
            assert np.array_equal(pts, ref["points"])
    finally:
        for s in ss:
            s.close()


@pytest.mark.parametrize("name", ["small_s3", "two_surface_24", "dense_12"])
def test_reconstruct_fft_background_matches_oracle(gpu, name):
    """background_mode = fft (reconstruct.hpp:405-429, denoise.hpp:267-319):
    the device FFT low-pass inside the tail stage against the oracle's direct
    DFT (<= 1e-9), through a whole reconstruction."""
    import dataclasses
    sc, cfg, _ = G.scene(name)
    cfg = dataclasses.replace(cfg, background_mode=1, fft_cutoff=0.4)
    gpu.set_scene(sc)
    rep = gpu.reconstruct(cfg)
    ref = O.reconstruct(sc, cfg, "oracle")
    assert rep["iterations"] == ref["iterations"]
    _assert_recon_parity(rep, ref, name + "/fft")
    np.testing.assert_allclose(rep["background"], ref["background"], rtol=1e-7, atol=1e-12)


@pytest.mark.parametrize("name", G.SCENE_NAMES)
def test_fused_and_separate_depth_block_agree(gpu, name):
    """The depth block run at the end of the previous stage kernel and as its
    own kernel give the same bits (reconstruct and palm_step flows)."""
    sc, cfg, _ = G.scene(name)
    a = _recon_with_env(gpu, sc, cfg, {})
    b = _recon_with_env(gpu, sc, cfg, {"RT3D_DEPTH_KERNEL": "1"})
    assert np.array_equal(a["points"], b["points"])
    assert np.array_equal(a["trace"], b["trace"])
    assert np.array_equal(a["steps"], b["steps"])


@pytest.mark.parametrize("name", G.SCENE_NAMES)
def test_one_launch_iteration_matches_kernel_sequence(gpu, name):
    """A PALM iteration as one cooperative launch (APSS, fit and kNN as grid
    phases) and as the kernel sequence give the same bits."""
    sc, cfg, _ = G.scene(name)
    a = _recon_with_env(gpu, sc, cfg, {})
    b = _recon_with_env(gpu, sc, cfg, {"RT3D_FUSED_ITER": "1"})
    assert np.array_equal(a["points"], b["points"])
    assert np.array_equal(a["background"], b["background"])
    assert np.array_equal(a["trace"], b["trace"])
    assert np.array_equal(a["steps"], b["steps"])


def _edge_scenes():
    import copy
    from scenegen.scene import SceneSpec, SurfaceSpec, simulate
    from paper_1905_06700_b200.abi import Config
    cfg = Config(max_iters=8, stop_tol=0.0, apss_radius=0.08, knn_k=9, r_min=0.25,
                 init_max_returns=3, init_peak_threshold=0.5, init_min_separation=6)
    dead = [(r, c) for r in range(0, 20, 3) for c in range(1, 20, 5)]
    spec = SceneSpec(rows=20, cols=20, bins=256, bin_resolution_m=0.01, pixel_pitch_m=0.02,
                     irf_sigma_bins=1.5, target_ppp=20.0, target_sbr=2.0, dead_pixels=dead,
                     surfaces=[SurfaceSpec(depth_m=1.0, holes=[(5, 5, 12, 12)]),
                               SurfaceSpec(depth_m=1.8)])
    holes = simulate(spec, 7)
    empty = copy.copy(holes)
    empty.offsets = np.zeros_like(holes.offsets)
    empty.events = holes.events[:0].copy()
    sparse = simulate(SceneSpec(rows=16, cols=16, bins=128, target_ppp=0.5, target_sbr=1.0,
                                surfaces=[SurfaceSpec(depth_m=0.6)]), 11)
    return {"dead_pixels_holes": (holes, cfg), "empty_cube": (empty, cfg),
            "sparse_half_photon": (sparse, cfg)}


@pytest.mark.parametrize("bg_mode", [0, 1])
@pytest.mark.parametrize("name", ["dead_pixels_holes", "empty_cube", "sparse_half_photon"])
def test_reconstruct_edge_cubes_match_oracle(gpu, name, bg_mode):
    """Ragged inputs the reference's tests exercise: dead (zero-event)
    pixels, an all-empty cube, and a cube at half a photon per pixel, with
    the identity and the FFT background.  The CUDA path and the C oracle
    agree (same tolerances as the golden scenes), and the streaming API
    (frame_submit / frame_collect) returns the same frame."""
    import dataclasses
    sc, cfg = _edge_scenes()[name]
    if bg_mode:
        cfg = dataclasses.replace(cfg, background_mode=1, fft_cutoff=0.4)
    gpu.set_scene(sc)
    rep = gpu.reconstruct(cfg)
    ref = O.reconstruct(sc, cfg, "oracle")
    assert rep["iterations"] == ref["iterations"]
    _assert_recon_parity(rep, ref, name)
    np.testing.assert_allclose(rep["background"], ref["background"],
                               rtol=1e-7 if bg_mode else 1e-9, atol=1e-12 if bg_mode else 1e-15)
    pts, bg, _ = gpu.frame_collect(gpu.frame_submit(sc, cfg))
    assert np.array_equal(pts, rep["points"])
    assert np.array_equal(bg, rep["background"])


@pytest.mark.parametrize("tol", [1e-3, 1e-5])
@pytest.mark.parametrize("name", ["two_surface_24", "small_s13", "dense_12"])
def test_reconstruct_early_stop_matches_oracle(gpu, name, tol):
    """stop_tol > 0: the relative-nll stopping rule (reconstruct.hpp's PALM
    loop) ends the device loop at the oracle's iteration, with the same
    cloud and trace."""
    import dataclasses
    sc, cfg, _ = G.scene(name)
    cfg = dataclasses.replace(cfg, stop_tol=tol, max_iters=40)
    ref = O.reconstruct(sc, cfg, "oracle")
    gpu.set_scene(sc)
    rep = gpu.reconstruct(cfg)
    assert rep["iterations"] == ref["iterations"], (rep["iterations"], ref["iterations"])
    _assert_recon_parity(rep, ref, f"{name}/tol{tol}")
    pts, bg, r2 = gpu.frame_collect(gpu.frame_submit(sc, cfg))
    assert np.array_equal(pts, rep["points"]) and r2["iterations"] == rep["iterations"]


@pytest.mark.parametrize("rows,cols", [(64, 64), (256, 256), (32, 128), (1024, 1024), (48, 64)])
def test_fft_lowpass_sizes(gpu, rows, cols):
    """fft_lowpass_filter (denoise.hpp:267-311) at power-of-two sizes (the
    radix-2 path) and a mixed one (the direct DFT) against the C oracle's
    direct DFT, relative to the image scale."""
    rng = np.random.default_rng(rows * 7 + cols)
    img = rng.uniform(0.0, 2.0, (rows, cols)) + np.outer(np.sin(np.arange(rows) / 5.0),
                                                        np.cos(np.arange(cols) / 7.0))
    for cutoff, clamp in ((0.3, False), (0.8, True), (1.0, False)):
        got = gpu.fft_lowpass(img, cutoff, clamp=clamp)
        if rows * cols <= 256 * 256:
            exp = O.fft_lowpass(img, cutoff, clamp=clamp, impl="oracle")
            assert np.max(np.abs(got - exp)) <= 1e-12 * np.max(np.abs(img)), (cutoff, clamp)
        else:   # the oracle's direct DFT is too slow here: linearity / identity properties
            if cutoff == 1.0:
                assert np.max(np.abs(got - img)) <= 1e-12 * np.max(np.abs(img))
            half = gpu.fft_lowpass(0.5 * img, cutoff, clamp=clamp)
            assert np.max(np.abs(2.0 * half - got)) <= 1e-12 * np.max(np.abs(img))


def test_apss_ball_overflow_matches_oracle(gpu):
    """Balls larger than the APSS member list (kApssCap, 208 per point): a dense
    two-surface scene with a radius of 12 fine pixels (~450 members per point)
    takes the chunk-by-chunk rescans (pass A and pass B) for most points, on
    both lane groups and through the shared pair scans; bit-identical to the
    oracle."""
    from paper_1905_06700_b200.abi import Config
    from scenegen.scene import SceneSpec, SurfaceSpec, simulate
    spec = SceneSpec(rows=32, cols=32, bins=300, bin_resolution_m=0.01, pixel_pitch_m=0.01,
                     target_ppp=20.0, target_sbr=5.0,
                     surfaces=[SurfaceSpec(depth_m=1.5), SurfaceSpec(depth_m=1.2, region=(8, 8, 24, 24))])
    cfg = Config(max_iters=3, stop_tol=0.0, apss_radius=0.12, knn_k=7, r_min=0.2,
                 init_max_returns=2, init_min_separation=6)
    sc = simulate(spec, 5)
    gpu.set_scene(sc)
    rep = gpu.reconstruct(cfg)
    ref = O.reconstruct(sc, cfg, "oracle")
    assert rep["iterations"] == ref["iterations"]
    assert np.array_equal(rep["points"], ref["points"])
    np.testing.assert_array_equal(rep["trace"], ref["trace"])
