"""Generate tests/golden/*.npz from the reference itself.

Run here (where /root/reference exists): `python tests/golden/make_golden.py`.
Inputs come from the reference's own generators — oracle::random_instance
(proj/tests/oracles.hpp:75-133) and simulate_cube (simulate.hpp:139-223) —
and the expected outputs from the reference headers compiled unchanged into
oracle/_ref/libref.so (test-only Eigen/FFTW stand-ins, see oracle/Makefile).
The fixtures are small so they can be committed; they let the GPU box, which
has no /root/reference, pin the oracle and the CUDA path to the reference.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))
sys.path.insert(0, str(HERE.parent))

import oracle_lib as L  # noqa: E402
from paper_1905_06700_b200.abi import Config  # noqa: E402

# SceneSpec texts (simulate.hpp:225-302 keys); presets mirror the reference
# tests: test_palm.cpp:15-40 (small), acceptance_main.cpp:50-80 (two-surface),
# test_init.cpp:299-334 (super-resolution), acceptance_main.cpp:262-289 (C6).
SMALL = """rows = 16
cols = 16
bins = 300
bin_resolution_m = 0.01
pixel_pitch_m = 0.02
irf_sigma_bins = 1.5
target_ppp = 6
target_sbr = 10
[surface]
depth_m = 1.5
"""
TWO_SURFACE_24 = """rows = 24
cols = 24
bins = 750
bin_resolution_m = 0.01
pixel_pitch_m = 0.02
irf_sigma_bins = 1.5
target_ppp = 3
target_sbr = 13
[surface]
depth_m = 7.0
[surface]
depth_m = 5.0
region = 6,6,18,18
"""
SUPERRES = """rows = 8
cols = 8
bins = 200
superres = 3
bin_resolution_m = 0.01
pixel_pitch_m = 0.05
irf_sigma_bins = 1.5
target_ppp = 15
target_sbr = 10
[surface]
depth_m = 1.0
slope_x = 0.5
"""
DENSE = """rows = 12
cols = 12
bins = 153
superres = 1
bin_resolution_m = 0.0375
pixel_pitch_m = 0.05
irf_sigma_bins = 1.5
target_ppp = 60
target_sbr = 1
[surface]
depth_m = 1.5
region = 0,0,12,6
[surface]
type = bump
depth_m = 3.0
bump_amp = -0.5
bump_cx = 0.3
bump_cy = 0.3
bump_width = 0.15
[surface]
depth_m = 4.5
"""

SMALL_CFG = dict(max_iters=5, apss_radius=0.1, knn_k=5, r_min=0.2, init_max_returns=2,
                 init_min_separation=6, stop_tol=0.0)
TWO_CFG = dict(max_iters=6, apss_radius=0.16, knn_k=9, r_min=0.25, init_max_returns=3,
               init_peak_threshold=0.5, init_min_separation=6, stop_tol=0.0)
SR_CFG = dict(max_iters=4, apss_radius=0.30, knn_k=9, r_min=0.2, init_max_returns=1,
              init_min_separation=6, stop_tol=0.0)
DENSE_CFG = dict(max_iters=4, apss_radius=0.16, knn_k=9, r_min=0.2, init_max_returns=3,
                 init_min_separation=6, stop_tol=0.0)

SCENES = {
    "small_s3": (SMALL, 3, SMALL_CFG),
    "small_s13": (SMALL, 13, SMALL_CFG),
    "two_surface_24": (TWO_SURFACE_24, 1234, TWO_CFG),
    "superres_8": (SUPERRES, 11, SR_CFG),
    "dense_12": (DENSE, 5, DENSE_CFG),
}


def scene_arrays(sc, prefix=""):
    d = {
        "rows": sc.n_rows, "cols": sc.n_cols, "bins": sc.n_bins, "superres": sc.superres,
        "pitch": sc.pixel_pitch, "bres": sc.bin_resolution, "bin_width_s": sc.bin_width_s,
        "offsets": sc.offsets, "events": sc.events.view(np.uint32).reshape(-1, 2),
        "irf": sc.irf_samples, "tau_min": sc.irf_tau_min, "dtau": sc.irf_dtau,
        "gain": sc.gain, "dead": sc.dead,
    }
    if sc.points is not None:
        d["points"] = sc.points
        d["background"] = sc.background
    return {prefix + k: np.asarray(v) for k, v in d.items()}


def evaluate_cases():
    """(name, est, truth, tau, pitch) for evaluate (eval.hpp:33-87): clouds with
    shared columns, equal depth errors (ties), negative coordinates, empties."""
    from paper_1905_06700_b200.abi import POINT_DTYPE
    rng = np.random.default_rng(1905)

    def cloud(n, span, zq=None, shift=0.0):
        c = np.zeros(n, POINT_DTYPE)
        c["x"] = rng.uniform(-span, span, n) + shift
        c["y"] = rng.uniform(-span, span, n)
        z = rng.uniform(1.0, 3.0, n)
        c["z"] = np.round(z / zq) * zq if zq else z
        c["intensity"] = rng.uniform(0.1, 5.0, n)
        return c

    cases = []
    sc = np.load(HERE / "scene_two_surface_24.npz")
    est = sc["rec_points"]
    truth = est.copy()
    truth["z"] += rng.normal(0, 0.01, len(truth))
    truth["intensity"] *= rng.uniform(0.8, 1.2, len(truth))
    keep = rng.random(len(truth)) > 0.1
    truth = np.concatenate([truth[keep], cloud(40, 0.2)])
    cases.append(("scene", est, truth, 0.02, float(sc["pitch"])))
    t = cloud(600, 0.05, zq=0.01)
    e = cloud(700, 0.05, zq=0.01)
    cases.append(("ties", e, t, 0.02, 0.01))
    cases.append(("ties_wide", e, t, 0.5, 0.02))
    e2 = cloud(300, 1.0, shift=-0.5)
    t2 = e2.copy()
    t2["z"] += rng.uniform(-0.05, 0.05, len(t2))
    cases.append(("negative", e2, t2, 0.03, 0.1))
    cases.append(("empty_est", e2[:0], t2, 0.03, 0.1))
    cases.append(("empty_truth", e2, t2[:0], 0.03, 0.1))
    cases.append(("empty_both", e2[:0], t2[:0], 0.03, 0.1))
    cases.append(("tiny_tau", e2, t2, 1e-12, 0.1))
    return cases


def make_evaluate():
    out = {}
    names = []
    for name, e, t, tau, pitch in evaluate_cases():
        r, rc = L.evaluate(e, t, tau, pitch, "ref")
        assert rc == 0, L.ref().ref_last_error()
        names.append(name)
        out[name + "_est"], out[name + "_truth"] = e, t
        out[name + "_tp"] = np.array([tau, pitch])
        out[name + "_out"] = r
    np.savez_compressed(HERE / "evaluate.npz", names=np.array(names), **out)
    print("evaluate cases", names)


def main():
    assert L.ref_available(), "oracle/_ref/libref.so missing: make -C oracle"
    if sys.argv[1:] == ["evaluate"]:
        make_evaluate()
        return
    # 1) random instances + reference likelihood outputs
    rnd = {}
    for seed in list(range(0, 40)) + [77, 9001, 1001, 1013]:
        dead = seed % 4 == 3 or seed == 77
        sc = L.ref_random_instance(seed, with_dead=dead)
        g = L.grads(sc, "ref")
        pre = f"r{seed}_"
        rnd.update(scene_arrays(sc, pre))
        rnd[pre + "nll"] = np.array(L.nll(sc, "ref"))
        rnd[pre + "dense_nll"] = np.array(L.ref().ref_dense_nll(*L.state_args(sc)))
        for k, v in g.items():
            rnd[pre + k] = v
    np.savez_compressed(HERE / "random_instances.npz", seeds=np.array(
        list(range(0, 40)) + [77, 9001, 1001, 1013]), **rnd)

    # 2) simulated scenes + reference init / palm_step / reconstruct
    for name, (text, seed, cfgd) in SCENES.items():
        cfg = Config(**cfgd)
        sc = L.ref_simulate(text, seed)
        out = scene_arrays(sc)
        out["cfg"] = np.array(repr(cfgd))
        pts, bg = L.init_matched_filter(sc, cfg, "ref")
        out["init_points"], out["init_background"] = pts, bg
        sc.with_state(pts, bg)
        p1, b1, d1 = L.palm_step(sc, cfg, "ref")
        out["palm_points"], out["palm_background"] = p1, b1
        out["palm_nll"] = np.array([d1.nll_before, d1.nll_after, d1.depth.nll_after_grad,
                                    d1.depth.nll_after_denoise, d1.intensity.nll_after_grad,
                                    d1.intensity.nll_after_denoise, d1.background.nll_after_grad])
        r = L.reconstruct(sc, cfg, "ref")
        out["rec_points"], out["rec_background"] = r["points"], r["background"]
        out["rec_trace"], out["rec_steps"] = r["trace"], r["steps"]
        out["baseline_points"] = L.baseline_xcorr(sc, "ref")
        np.savez_compressed(HERE / f"scene_{name}.npz", **out)
        print(name, "events", len(sc.events), "init pts", len(pts), "rec pts",
              len(r["points"]), "iters", r["iterations"])

    # 3) reference matched-filter peaks on a few hand-made pixels
    irf, tmin = L.irf_gaussian(1.5)
    sc = L.ref_random_instance(3)
    peaks = {}
    cases = {
        "sym": [(99, 3), (100, 5), (101, 3)],
        "two": [(20, 4), (21, 6), (60, 1), (70, 1), (80, 1), (90, 1), (95, 1)],
        "edge": [(0, 2), (1, 3), (198, 1), (199, 4)],
        "ties": [(10, 1), (30, 1), (50, 1), (70, 1)],
    }
    from paper_1905_06700_b200.abi import EVENT_DTYPE, Scene
    one = Scene(1, 1, 200, np.array([0, 0], np.uint64), np.zeros(0, EVENT_DTYPE), irf, tmin, 0.25)
    for name, evs in cases.items():
        ev = np.array(evs, np.uint32).view(EVENT_DTYPE).reshape(-1)
        for (k, thr, sep) in [(3, 0.5, 3), (1, 0.0, 1), (2, 1.0, 10), (4, 0.5, 1)]:
            pk = L.matched_filter_peaks(ev, one, k, thr, sep, "ref")
            peaks[f"{name}_{k}_{thr}_{sep}_events"] = np.array(evs, np.uint32)
            peaks[f"{name}_{k}_{thr}_{sep}"] = pk
    peaks["irf"], peaks["tau_min"] = irf, tmin
    np.savez_compressed(HERE / "peaks.npz", **peaks)

    # 4) reference APSS / kNN / FFT on the denoise tests' clouds
    rng = np.random.default_rng(12345)
    from paper_1905_06700_b200.abi import POINT_DTYPE

    def cloud(xyz, inten=None):
        p = np.zeros(len(xyz), POINT_DTYPE)
        p["x"], p["y"], p["z"] = xyz.T
        p["intensity"] = rng.random(len(xyz)) * 4 if inten is None else inten
        return p

    n = 300
    u = 2 * rng.random(n) - 1
    phi = 2 * np.pi * rng.random(n)
    s = np.sqrt(1 - u * u)
    sph = cloud(np.array([2.0, -1.0, 5.0]) + np.stack([s * np.cos(phi), s * np.sin(phi), u], 1))
    noisy = cloud(np.stack([2 * rng.random(600), 2 * rng.random(600),
                            0.02 * rng.standard_normal(600)], 1))
    den = {"sphere": sph, "noisy": noisy,
           "sphere_apss": L.apss_project(sph, 0.45, impl="ref"),
           "noisy_apss": L.apss_project(noisy, 0.2, impl="ref"),
           "noisy_knn6": L.knn_filter(noisy, 6, 0.25, impl="ref"),
           "noisy_knn1": L.knn_filter(noisy, 1, 0.25, impl="ref")}
    img = rng.random((14, 17))
    den["img"] = img
    den["img_fft04"] = L.fft_lowpass(img, 0.4, impl="ref")
    den["img_fft04_clamp"] = L.fft_lowpass(img, 0.4, clamp=True, impl="ref")
    np.savez_compressed(HERE / "denoise.npz", **den)
    make_evaluate()
    print("done")


if __name__ == "__main__":
    main()
