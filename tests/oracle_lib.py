"""Test-side bindings for the checkers: oracle/liboracle.so (the C
restatement) and oracle/_ref/libref.so (the reference headers compiled
unchanged with test-only Eigen/FFTW stand-ins).  Only tests/, smoke() and
bench.py's cpu_baseline leg use this module.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path
from typing import Optional

import numpy as np

from paper_1905_06700_b200.abi import (
    EVENT_DTYPE, POINT_DTYPE, PEAK_DTYPE, STEP_DIAG_DTYPE, ApssParams, Cube, Event, InitParams,
    Irf, Peak, Point, ReconConfig, Scene, Sensor, StepDiag, ptr,
)

ROOT = Path(__file__).resolve().parents[1]
ORACLE_SO = ROOT / "oracle" / "liboracle.so"
REF_SO = ROOT / "oracle" / "_ref" / "libref.so"

P = C.POINTER
_dbl, _u64, _u8, _i32 = C.c_double, C.c_uint64, C.c_uint8, C.c_int32


def _bind(lib, name, res, args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = args
    return f


class _Lib:
    """Common wrappers over the oracle_* / ref_* C functions."""

    def __init__(self, path: Path, prefix: str):
        self.lib = C.CDLL(str(path))
        self.prefix = prefix

    def fn(self, name):
        return getattr(self.lib, self.prefix + name)


_oracle: Optional[C.CDLL] = None
_ref: Optional[C.CDLL] = None


def oracle() -> C.CDLL:
    global _oracle
    if _oracle is None:
        if not ORACLE_SO.exists():
            raise RuntimeError(f"{ORACLE_SO} missing: run `make -C oracle`")
        lib = C.CDLL(str(ORACLE_SO))
        _bind(lib, "oracle_irf_gaussian", _u64, [_dbl, _dbl, _dbl, P(_dbl), _u64, P(_dbl)])
        _bind(lib, "oracle_irf_value", _dbl, [P(Irf), _dbl])
        _bind(lib, "oracle_irf_deriv", _dbl, [P(Irf), _dbl])
        _bind(lib, "oracle_irf_mass_in_gate", _dbl, [P(Irf), _dbl, C.c_int])
        _bind(lib, "oracle_pairwise_sum", _dbl, [P(_dbl), _u64])
        _bind(lib, "oracle_matched_filter_peaks", C.c_int,
              [P(Event), _u64, P(Irf), C.c_int, C.c_int, _dbl, C.c_int, P(Peak)])
        _bind(lib, "oracle_init_matched_filter", C.c_int,
              [P(Cube), P(Sensor), P(InitParams), P(Point), P(_u64), P(_dbl)])
        _bind(lib, "oracle_nll", _dbl, [P(Cube), P(Sensor), P(Point), _u64, P(_dbl)])
        for nm in ("oracle_grad_intensity", "oracle_grad_background"):
            _bind(lib, nm, None, [P(Cube), P(Sensor), P(Point), _u64, P(_dbl), P(_dbl)])
        _bind(lib, "oracle_grad_depth", None,
              [P(Cube), P(Sensor), P(Point), _u64, P(_dbl), P(_dbl), P(_u8)])
        _bind(lib, "oracle_block_curvatures", None,
              [P(Cube), P(Sensor), P(Point), _u64, P(_dbl), P(_dbl), P(_dbl), P(_dbl)])
        _bind(lib, "oracle_apss_project", C.c_int,
              [P(Point), _u64, P(ApssParams), P(Point), _u64, _dbl, P(Point)])
        _bind(lib, "oracle_knn_intensity_filter", C.c_int,
              [P(Point), _u64, C.c_int, P(Point), _u64, _dbl, _dbl, P(Point)])
        _bind(lib, "oracle_prune", _u64, [P(Point), _u64, _dbl, P(Point)])
        _bind(lib, "oracle_evaluate", C.c_int, [P(Point), _u64, P(Point), _u64, _dbl, _dbl, P(_dbl)])
        _bind(lib, "oracle_fft_lowpass_filter", C.c_int,
              [P(_dbl), C.c_int, C.c_int, _dbl, C.c_int, P(_dbl)])
        _bind(lib, "oracle_palm_step", C.c_int,
              [P(Cube), P(Sensor), P(ReconConfig), P(Point), P(_u64), P(_dbl), P(StepDiag)])
        _bind(lib, "oracle_reconstruct", C.c_int,
              [P(Cube), P(Sensor), P(ReconConfig), P(Point), P(_u64), P(_dbl), P(_dbl),
               P(StepDiag), P(C.c_int)])
        _bind(lib, "oracle_baseline_xcorr", C.c_int,
              [P(Cube), P(Sensor), P(Point), P(_u64)])
        _bind(lib, "oracle_pratt_smallest", C.c_int, [P(_dbl), P(_dbl)])
        _bind(lib, "oracle_sym3_eigenvalues", None, [P(_dbl), P(_dbl)])
        _oracle = lib
    return _oracle


def ref_available() -> bool:
    return REF_SO.exists()


def ref() -> C.CDLL:
    global _ref
    if _ref is None:
        lib = C.CDLL(str(REF_SO))
        _bind(lib, "ref_last_error", C.c_char_p, [])
        _bind(lib, "ref_set_threads", None, [C.c_uint])
        _bind(lib, "ref_matched_filter_peaks", C.c_int,
              [P(Event), _u64, P(Irf), C.c_int, C.c_int, _dbl, C.c_int, P(Peak)])
        _bind(lib, "ref_init_matched_filter", C.c_int,
              [P(Cube), P(Sensor), P(InitParams), P(Point), P(_u64), P(_dbl)])
        _bind(lib, "ref_nll", _dbl, [P(Cube), P(Sensor), P(Point), _u64, P(_dbl)])
        _bind(lib, "ref_dense_nll", _dbl, [P(Cube), P(Sensor), P(Point), _u64, P(_dbl)])
        _bind(lib, "ref_grads", C.c_int,
              [P(Cube), P(Sensor), P(Point), _u64, P(_dbl), P(_dbl), P(_u8), P(_dbl), P(_dbl),
               P(_dbl), P(_dbl), P(_dbl)])
        _bind(lib, "ref_apss_project", C.c_int, [P(Point), _u64, P(ApssParams), _dbl, P(Point)])
        _bind(lib, "ref_knn_intensity_filter", C.c_int,
              [P(Point), _u64, C.c_int, _dbl, _dbl, P(Point)])
        _bind(lib, "ref_fft_lowpass", C.c_int, [P(_dbl), C.c_int, C.c_int, _dbl, C.c_int, P(_dbl)])
        _bind(lib, "ref_palm_step", C.c_int,
              [P(Cube), P(Sensor), P(ReconConfig), P(Point), P(_u64), P(_dbl), P(StepDiag)])
        _bind(lib, "ref_reconstruct_full", C.c_int,
              [P(Cube), P(Sensor), P(ReconConfig), P(Point), P(_u64), P(_dbl), P(_dbl),
               P(StepDiag), P(C.c_int)])
        _bind(lib, "ref_reconstruct", C.c_int,
              [P(Cube), P(Sensor), P(ReconConfig), P(_u64), P(C.c_int), P(_dbl)])
        _bind(lib, "ref_result_copy", C.c_int, [P(Point), P(_dbl)])
        _bind(lib, "ref_evaluate", C.c_int, [P(Point), _u64, P(Point), _u64, _dbl, _dbl, P(_dbl)])
        _bind(lib, "ref_baseline_xcorr", C.c_int, [P(Cube), P(Sensor), P(Point), P(_u64)])
        _bind(lib, "ref_simulate", C.c_int,
              [C.c_char_p, _u64, P(C.c_int), P(_u64), P(_u64)])
        _bind(lib, "ref_random_instance", C.c_int,
              [_u64, C.c_int, P(C.c_int), P(_u64), P(_u64)])
        _bind(lib, "ref_held_copy", C.c_int,
              [P(_u64), P(Event), P(_dbl), P(_u8), P(_dbl), P(_dbl), P(Point), P(_dbl)])
        _bind(lib, "ref_irf_gaussian", _u64, [_dbl, _dbl, _dbl, P(_dbl), P(_dbl)])
        _ref = lib
    return _ref


# ---------------------------------------------------------------------------
# inputs produced by the reference itself
# ---------------------------------------------------------------------------
def _held_scene(dims, n_events, n_points, with_state: bool) -> Scene:
    lib = ref()
    rows, cols, bins, s = dims
    npix = rows * cols
    offsets = np.zeros(npix + 1, np.uint64)
    events = np.zeros(max(n_events, 1), EVENT_DTYPE)
    gain = np.zeros(npix)
    dead = np.zeros(npix, np.uint8)
    meta = np.zeros(6)
    irf = np.zeros(4096)
    pts = np.zeros(max(n_points, 1), POINT_DTYPE)
    bg = np.zeros(npix)
    lib.ref_held_copy(ptr(offsets, _u64), ptr(events, Event), ptr(gain, _dbl), ptr(dead, _u8),
                      ptr(irf, _dbl), ptr(meta, _dbl), ptr(pts, Point),
                      ptr(bg, _dbl) if with_state else None)
    n_irf = int(meta[2])
    sc = Scene(rows, cols, bins, offsets, events[:n_events], irf[:n_irf].copy(), meta[0],
               meta[1], superres=s, pixel_pitch=meta[3], bin_resolution=meta[4],
               bin_width_s=meta[5], gain=gain, dead=dead)
    if with_state:
        sc.with_state(pts[:n_points].copy(), bg)
    else:
        sc.truth = pts[:n_points].copy()
    return sc


def ref_random_instance(seed: int, with_dead: bool = False) -> Scene:
    """oracle::random_instance from the reference's tests/oracles.hpp:75-133."""
    dims = (C.c_int * 4)()
    ne, npn = _u64(), _u64()
    rc = ref().ref_random_instance(seed, int(with_dead), dims, C.byref(ne), C.byref(npn))
    assert rc == 0, ref().ref_last_error()
    return _held_scene(tuple(dims), ne.value, npn.value, True)


def ref_simulate(scene_text: str, seed: int) -> Scene:
    """simulate_cube on a SceneSpec key=value text (simulate.hpp:139-302)."""
    dims = (C.c_int * 4)()
    ne, nt = _u64(), _u64()
    rc = ref().ref_simulate(scene_text.encode(), seed, dims, C.byref(ne), C.byref(nt))
    assert rc == 0, ref().ref_last_error()
    return _held_scene(tuple(dims), ne.value, nt.value, False)


# ---------------------------------------------------------------------------
# uniform calls on either checker: impl is "oracle" or "ref"
# ---------------------------------------------------------------------------
def _lib(impl):
    return oracle() if impl == "oracle" else ref()


def _name(impl, op):
    return ("oracle_" if impl == "oracle" else "ref_") + op


def state_args(sc: Scene):
    return (C.byref(sc.cube_c()), C.byref(sc.sensor_c()), ptr(sc.points, Point),
            len(sc.points), ptr(sc.background, _dbl))


def nll(sc: Scene, impl="oracle") -> float:
    return getattr(_lib(impl), _name(impl, "nll"))(*state_args(sc))


def grads(sc: Scene, impl="oracle"):
    n, npix = len(sc.points), sc.n_pixels
    out = {k: np.zeros(n) for k in ("gd", "gr", "cd", "cr")}
    out["oog"] = np.zeros(n, np.uint8)
    out["gb"] = np.zeros(npix)
    out["cb"] = np.zeros(npix)
    if impl == "ref":
        rc = ref().ref_grads(*state_args(sc), ptr(out["gd"], _dbl), ptr(out["oog"], _u8),
                             ptr(out["gr"], _dbl), ptr(out["gb"], _dbl), ptr(out["cd"], _dbl),
                             ptr(out["cr"], _dbl), ptr(out["cb"], _dbl))
        assert rc == 0, ref().ref_last_error()
    else:
        o = oracle()
        gdn = np.zeros(n) if n == 0 else out["gd"]
        o.oracle_grad_depth(*state_args(sc), ptr(out["gd"], _dbl), ptr(out["oog"], _u8))
        o.oracle_grad_intensity(*state_args(sc), ptr(out["gr"], _dbl))
        o.oracle_grad_background(*state_args(sc), ptr(out["gb"], _dbl))
        o.oracle_block_curvatures(*state_args(sc), ptr(out["cd"], _dbl), ptr(out["cr"], _dbl),
                                  ptr(out["cb"], _dbl))
        del gdn
    return out


def init_matched_filter(sc: Scene, cfg, impl="oracle"):
    cap = max(1, cfg.init_max_returns * sc.superres ** 2 * sc.n_pixels)
    pts = np.zeros(cap, POINT_DTYPE)
    bg = np.zeros(sc.n_pixels)
    n = _u64()
    ip = cfg.init_c()
    rc = getattr(_lib(impl), _name(impl, "init_matched_filter"))(
        C.byref(sc.cube_c()), C.byref(sc.sensor_c()), C.byref(ip), ptr(pts, Point), C.byref(n),
        ptr(bg, _dbl))
    assert rc == 0
    return pts[: n.value].copy(), bg


def matched_filter_peaks(events, sc: Scene, k, thr, min_sep, impl="oracle"):
    events = np.ascontiguousarray(events, EVENT_DTYPE)
    out = np.zeros(max(k, 1), PEAK_DTYPE)
    irf = sc.irf_c()
    fn = getattr(_lib(impl), _name(impl, "matched_filter_peaks"))
    cnt = fn(ptr(events, Event) if len(events) else None, len(events), C.byref(irf), sc.n_bins, k,
             thr, min_sep, out.ctypes.data_as(P(Peak)))
    return out[:cnt].copy()


def palm_step(sc: Scene, cfg, impl="oracle"):
    pts = sc.points.copy()
    bg = sc.background.copy()
    n = _u64(len(pts))
    d = StepDiag()
    c = cfg.to_c()
    rc = getattr(_lib(impl), _name(impl, "palm_step"))(
        C.byref(sc.cube_c()), C.byref(sc.sensor_c()), C.byref(c), ptr(pts, Point), C.byref(n),
        ptr(bg, _dbl), C.byref(d))
    assert rc == 0
    return pts[: n.value].copy(), bg, d


def reconstruct(sc: Scene, cfg, impl="oracle"):
    cap = max(1, cfg.init_max_returns * sc.superres ** 2 * sc.n_pixels)
    pts = np.zeros(cap, POINT_DTYPE)
    bg = np.zeros(sc.n_pixels)
    trace = np.zeros(cfg.max_iters + 1)
    steps = np.zeros(cfg.max_iters, STEP_DIAG_DTYPE)
    n = _u64()
    it = C.c_int()
    c = cfg.to_c()
    fn = "oracle_reconstruct" if impl == "oracle" else "ref_reconstruct_full"
    rc = getattr(_lib(impl), fn)(
        C.byref(sc.cube_c()), C.byref(sc.sensor_c()), C.byref(c), ptr(pts, Point), C.byref(n),
        ptr(bg, _dbl), ptr(trace, _dbl), steps.ctypes.data_as(P(StepDiag)), C.byref(it))
    assert rc == 0
    return dict(points=pts[: n.value].copy(), background=bg, trace=trace[: it.value + 1],
                steps=steps[: it.value], iterations=it.value)


def apss_project(points, radius, min_nbrs=6, eps=1e-3, cell=None, impl="oracle"):
    points = np.ascontiguousarray(points, POINT_DTYPE)
    out = np.zeros(len(points), POINT_DTYPE)
    ap = ApssParams()
    ap.kernel_radius, ap.min_neighbors, ap.sphere_degeneracy_eps = radius, min_nbrs, eps
    cell = radius if cell is None else cell
    if impl == "oracle":
        rc = oracle().oracle_apss_project(ptr(points, Point), len(points), C.byref(ap),
                                          ptr(points, Point), len(points), cell, ptr(out, Point))
    else:
        rc = ref().ref_apss_project(ptr(points, Point), len(points), C.byref(ap), cell,
                                    ptr(out, Point))
    assert rc == 0
    return out


def knn_filter(points, k, radius, cell=None, impl="oracle"):
    points = np.ascontiguousarray(points, POINT_DTYPE)
    out = np.zeros(len(points), POINT_DTYPE)
    cell = radius if cell is None else cell
    if impl == "oracle":
        rc = oracle().oracle_knn_intensity_filter(ptr(points, Point), len(points), k,
                                                  ptr(points, Point), len(points), cell, radius,
                                                  ptr(out, Point))
    else:
        rc = ref().ref_knn_intensity_filter(ptr(points, Point), len(points), k, cell, radius,
                                            ptr(out, Point))
    assert rc == 0
    return out


def fft_lowpass(img, cutoff, clamp=False, impl="oracle"):
    img = np.ascontiguousarray(img, np.float64)
    out = np.zeros_like(img)
    fn = "oracle_fft_lowpass_filter" if impl == "oracle" else "ref_fft_lowpass"
    rc = getattr(_lib(impl), fn)(ptr(img, _dbl), img.shape[0], img.shape[1], cutoff, int(clamp),
                                 ptr(out, _dbl))
    return out if rc == 0 else None


def baseline_xcorr(sc: Scene, impl="oracle"):
    pts = np.zeros(max(1, sc.n_pixels), POINT_DTYPE)
    n = _u64()
    rc = getattr(_lib(impl), _name(impl, "baseline_xcorr"))(
        C.byref(sc.cube_c()), C.byref(sc.sensor_c()), ptr(pts, Point), C.byref(n))
    assert rc == 0
    return pts[: n.value].copy()


def irf_gaussian(sigma=1.5, nsig=4.0, dtau=0.25):
    buf = np.zeros(4096)
    tmin = _dbl()
    n = oracle().oracle_irf_gaussian(sigma, nsig, dtau, ptr(buf, _dbl), len(buf), C.byref(tmin))
    return buf[:n].copy(), tmin.value


def evaluate(est, truth, tau: float, pitch: float, impl="oracle"):
    """eval.hpp:33-87 -> (7 doubles, status): recall, false_point_rate, depth_rmse,
    intensity_mae, n_truth, n_est, n_matched."""
    est = np.ascontiguousarray(est, POINT_DTYPE)
    truth = np.ascontiguousarray(truth, POINT_DTYPE)
    out = np.zeros(7)
    rc = getattr(_lib(impl), _name(impl, "evaluate"))(ptr(est, Point), len(est), ptr(truth, Point),
                                                       len(truth), tau, pitch, ptr(out, _dbl))
    return out, rc
