"""ctypes binding of librt3d.so (include/rt3d.h).

The library is built in-tree (paper_1905_06700_b200/librt3d.so) by
__graft_entry__.build().  Loading fails loudly when it is missing, and every
compute call raises when no CUDA device is present: there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path
from typing import Optional

import numpy as np

from .abi import (
    EVENT_DTYPE, POINT_DTYPE, PEAK_DTYPE, STEP_DIAG_DTYPE, STATUS, ApssParams, Cube, Event, InitParams, Irf,
    Peak, Point, ReconConfig, Report, Scene, Sensor, StateView, StepDiag, Config, ptr,
)

LIB_PATH = Path(os.environ.get("RT3D_LIB", Path(__file__).resolve().parent / "librt3d.so"))

P = C.POINTER
_dbl, _u64, _u8, _i32, _st = C.c_double, C.c_uint64, C.c_uint8, C.c_int32, C.c_int


class Rt3dError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"rt3d {STATUS.get(status, status)}: {msg}")
        self.status = status


_lib: Optional[C.CDLL] = None


def _bind(lib, name, res, args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = args


def lib() -> C.CDLL:
    """Load librt3d.so (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() first")
    L = C.CDLL(str(LIB_PATH))
    SS = C.c_void_p
    _bind(L, "rt3d_abi_version", C.c_int, [])
    _bind(L, "rt3d_last_error", C.c_char_p, [])
    _bind(L, "rt3d_device_count", C.c_int, [])
    _bind(L, "rt3d_session_create", _st, [C.c_int, P(SS)])
    _bind(L, "rt3d_session_destroy", _st, [SS])
    _bind(L, "rt3d_session_synchronize", _st, [SS])
    _bind(L, "rt3d_session_set_sharing", _st, [SS, C.c_int])
    _bind(L, "rt3d_session_after", _st, [SS, SS])
    _bind(L, "rt3d_session_stream", C.c_void_p, [SS])
    _bind(L, "rt3d_session_profile", _st, [SS, C.c_int])
    _bind(L, "rt3d_profile_copy", _st, [SS, P(_u64), C.c_uint32, P(C.c_uint32)])
    _bind(L, "rt3d_session_time_kernels", _st, [SS, C.c_int])
    _bind(L, "rt3d_kernel_times", _st, [SS, P(_dbl), P(_u64)])
    _bind(L, "rt3d_graph_counts", _st, [SS, P(_u64), P(_u64)])
    _bind(L, "rt3d_debug_buffer", C.c_void_p, [SS])
    _bind(L, "rt3d_set_sensor", _st, [SS, P(Sensor)])
    _bind(L, "rt3d_set_cube", _st, [SS, P(Cube)])
    _bind(L, "rt3d_set_cube_spcb", _st, [SS, C.c_void_p, _u64])
    _bind(L, "rt3d_reconstruct", _st, [SS, P(ReconConfig)])
    _bind(L, "rt3d_reconstruct_batch", _st, [P(SS), _i32, P(ReconConfig)])
    _bind(L, "rt3d_reconstruct_bands", _st, [P(SS), _i32, P(ReconConfig)])
    _bind(L, "rt3d_band_pixels", _st, [SS, P(C.c_uint32), P(C.c_uint32)])
    _bind(L, "rt3d_measure_fp64_peak", _st, [SS, P(_dbl)])
    _bind(L, "rt3d_band_plan", _st, [C.c_uint32, C.c_uint32, _i32, _dbl, _dbl, _i32,
                                     P(C.c_uint32), P(C.c_uint32), P(C.c_uint32)])
    _bind(L, "rt3d_frame_submit", _st, [SS, P(Cube), P(ReconConfig), P(_u64)])
    _bind(L, "rt3d_frame_collect", _st, [SS, _u64, P(Point), _u64, P(_u64), P(_dbl), P(Report)])
    _bind(L, "rt3d_report_info", _st, [SS, P(Report)])
    _bind(L, "rt3d_report_copy", _st, [SS, P(_dbl), P(StepDiag)])
    _bind(L, "rt3d_state_size", _st, [SS, P(_u64)])
    _bind(L, "rt3d_state_copy", _st, [SS, P(Point), P(_dbl)])
    _bind(L, "rt3d_matched_filter_peaks", _st,
          [SS, P(Event), _u64, P(Irf), _i32, _i32, _dbl, _i32, P(Peak), P(_i32)])
    _bind(L, "rt3d_init_matched_filter", _st, [SS, P(InitParams)])
    _bind(L, "rt3d_baseline_xcorr", _st, [SS])
    _bind(L, "rt3d_state_upload", _st, [SS, P(StateView)])
    _bind(L, "rt3d_nll", _st, [SS, P(_dbl)])
    _bind(L, "rt3d_grad_depth", _st, [SS, P(_dbl), P(_u8)])
    _bind(L, "rt3d_grad_intensity", _st, [SS, P(_dbl)])
    _bind(L, "rt3d_grad_background", _st, [SS, P(_dbl)])
    _bind(L, "rt3d_block_curvatures", _st, [SS, P(_dbl), P(_dbl), P(_dbl)])
    _bind(L, "rt3d_palm_step", _st, [SS, P(ReconConfig), P(StepDiag)])
    _bind(L, "rt3d_apss_project", _st,
          [SS, P(Point), _u64, P(ApssParams), P(Point), _u64, _dbl, P(Point)])
    _bind(L, "rt3d_knn_intensity_filter", _st,
          [SS, P(Point), _u64, _i32, P(Point), _u64, _dbl, _dbl, P(Point)])
    _bind(L, "rt3d_prune", _st, [SS, P(Point), _u64, _dbl, P(Point), P(_u64)])
    _bind(L, "rt3d_evaluate", _st, [SS, P(Point), _u64, P(Point), _u64, _dbl, _dbl, P(Eval)])
    _bind(L, "rt3d_fft_lowpass_filter", _st,
          [SS, P(_dbl), _i32, _i32, _dbl, _i32, P(_dbl)])
    _bind(L, "rt3d_simulate_cube", _st, [SS, P(Point), _u64, P(_dbl), _u64, P(_u64), P(_u64)])
    _bind(L, "rt3d_cube_copy", _st, [SS, P(_u64), P(Event)])
    _bind(L, "rt3d_encode_ply", _st, [P(Point), _u64, _i32, _dbl, C.c_char_p, _u64, P(_u64)])
    _bind(L, "rt3d_encode_background_csv", _st, [P(_dbl), _i32, _i32, C.c_char_p, _u64, P(_u64)])
    _lib = L
    return L


def _check(status: int):
    if status != 0:
        raise Rt3dError(status, lib().rt3d_last_error().decode(errors="replace"))


EXPORTED = [
    "rt3d_abi_version", "rt3d_last_error", "rt3d_device_count", "rt3d_session_create",
    "rt3d_session_destroy", "rt3d_session_synchronize", "rt3d_session_set_sharing", "rt3d_session_after", "rt3d_session_stream", "rt3d_session_profile", "rt3d_profile_copy",
    "rt3d_session_time_kernels", "rt3d_kernel_times", "rt3d_graph_counts", "rt3d_debug_buffer",
    "rt3d_set_sensor", "rt3d_set_cube", "rt3d_set_cube_spcb",
    "rt3d_reconstruct", "rt3d_reconstruct_batch", "rt3d_reconstruct_bands", "rt3d_band_pixels",
    "rt3d_band_plan", "rt3d_measure_fp64_peak",
    "rt3d_frame_submit", "rt3d_frame_collect", "rt3d_report_info", "rt3d_report_copy", "rt3d_state_size",
    "rt3d_state_copy", "rt3d_matched_filter_peaks", "rt3d_init_matched_filter",
    "rt3d_baseline_xcorr", "rt3d_state_upload", "rt3d_nll", "rt3d_grad_depth",
    "rt3d_grad_intensity", "rt3d_grad_background", "rt3d_block_curvatures", "rt3d_palm_step",
    "rt3d_apss_project", "rt3d_knn_intensity_filter", "rt3d_prune", "rt3d_fft_lowpass_filter",
    "rt3d_evaluate", "rt3d_encode_ply", "rt3d_encode_background_csv",
    "rt3d_simulate_cube", "rt3d_cube_copy",
]


def band_plan(rows: int, cols: int, superres: int, pixel_pitch: float, apss_radius: float, n: int):
    """rt3d_band_plan (host only): ([(begin, end)] pixel ranges of the n row
    bands, halo rows read on either side)."""
    b = (C.c_uint32 * n)()
    e = (C.c_uint32 * n)()
    h = C.c_uint32()
    _check(lib().rt3d_band_plan(rows, cols, superres, pixel_pitch, apss_radius, n, b, e,
                                C.byref(h)))
    return [(int(b[k]), int(e[k])) for k in range(n)], int(h.value)


def _two_call(fn, *args) -> bytes:
    n = _u64()
    _check(fn(*args, None, 0, C.byref(n)))
    buf = C.create_string_buffer(max(n.value, 1))
    _check(fn(*args, buf, n.value, C.byref(n)))
    return buf.raw[: n.value]


def encode_ply(points, pixel_pitch=None) -> bytes:
    """encode_ply (io.hpp:162-179): the reference's ASCII PLY bytes."""
    points = np.ascontiguousarray(points, POINT_DTYPE)
    return _two_call(lib().rt3d_encode_ply, ptr(points, Point), len(points),
                     int(pixel_pitch is not None), float(pixel_pitch or 0.0))


def encode_background_csv(background) -> bytes:
    """`splidar reconstruct --background-out` CSV (tools/splidar_main.cpp:204-212)."""
    bg = np.ascontiguousarray(background, np.float64)
    rows, cols = bg.shape
    return _two_call(lib().rt3d_encode_background_csv, ptr(bg, _dbl), rows, cols)


class Eval(C.Structure):
    """rt3d_eval (include/rt3d.h) = splidar::EvalResult (eval.hpp:21-29)."""
    _fields_ = [("recall", C.c_double), ("false_point_rate", C.c_double),
                ("depth_rmse", C.c_double), ("intensity_mae", C.c_double),
                ("n_truth", C.c_uint64), ("n_est", C.c_uint64), ("n_matched", C.c_uint64)]


class Session:
    """One CUDA device + stream with resident sensor / cube / state."""

    def __init__(self, device: int = 0):
        L = lib()
        h = C.c_void_p()
        _check(L.rt3d_session_create(device, C.byref(h)))
        self.h = h
        self.scene: Optional[Scene] = None

    def close(self):
        if self.h:
            lib().rt3d_session_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- inputs ----------------------------------------------------------
    def set_scene(self, sc: Scene):
        L = lib()
        self._sensor = sc.sensor_c()
        self._cube = sc.cube_c()
        _check(L.rt3d_set_sensor(self.h, C.byref(self._sensor)))
        _check(L.rt3d_set_cube(self.h, C.byref(self._cube)))
        self.scene = sc

    def set_cube(self, sc: Scene):
        self._cube = sc.cube_c()
        _check(lib().rt3d_set_cube(self.h, C.byref(self._cube)))

    def set_cube_spcb(self, data):
        """decode_cube (io.hpp:116-145) of SPCB bytes into the device CSR."""
        buf = np.frombuffer(bytes(data), np.uint8) if not isinstance(data, np.ndarray) else data
        buf = np.ascontiguousarray(buf, np.uint8)
        _check(lib().rt3d_set_cube_spcb(self.h, buf.ctypes.data if len(buf) else None, len(buf)))

    def upload_state(self, points: np.ndarray, background: np.ndarray):
        from .abi import buckets
        sc = self.scene
        points = np.ascontiguousarray(points, POINT_DTYPE)
        background = np.ascontiguousarray(background, np.float64)
        bo, bp = buckets(points, sc.n_rows, sc.n_cols)
        v = StateView()
        v.points = ptr(points, Point) if len(points) else None
        v.n_points = len(points)
        v.background = ptr(background, _dbl)
        v.bucket_offsets = ptr(bo, C.c_uint32)
        v.bucket_points = ptr(bp, C.c_uint32) if len(points) else None
        self._keep = (points, background, bo, bp)
        _check(lib().rt3d_state_upload(self.h, C.byref(v)))

    # -- hot path --------------------------------------------------------
    def reconstruct_async(self, cfg: Config):
        self._cfg_c = cfg.to_c()
        _check(lib().rt3d_reconstruct(self.h, C.byref(self._cfg_c)))

    @staticmethod
    def reconstruct_batch_async(sessions, cfg: Config):
        """rt3d_reconstruct_batch: one frame per session (each on its own
        resident cube) in one launch sequence on sessions[0]'s stream."""
        arr = (C.c_void_p * len(sessions))(*[s.h for s in sessions])
        c = cfg.to_c()
        sessions[0]._cfg_c = c
        _check(lib().rt3d_reconstruct_batch(arr, len(sessions), C.byref(c)))

    @staticmethod
    def reconstruct_bands(sessions, cfg: Config) -> dict:
        """rt3d_reconstruct_bands: one frame split into len(sessions) row
        bands (every session holds the same sensor and cube); returns the
        frame's cloud (the bands' clouds in order), background and report."""
        arr = (C.c_void_p * len(sessions))(*[s.h for s in sessions])
        c = cfg.to_c()
        _check(lib().rt3d_reconstruct_bands(arr, len(sessions), C.byref(c)))
        rep = sessions[0].report()
        parts, bg = [], None
        for s in sessions:
            pts, b = s.state()
            a, z = C.c_uint32(), C.c_uint32()
            _check(lib().rt3d_band_pixels(s.h, C.byref(a), C.byref(z)))
            if bg is None:
                bg = np.zeros_like(b)
            bg[a.value:z.value] = b[a.value:z.value]
            parts.append(pts)
        rep["points"] = np.concatenate(parts) if parts else np.zeros(0, POINT_DTYPE)
        rep["background"] = bg
        return rep

    @property
    def stream_ptr(self) -> int:
        return lib().rt3d_session_stream(self.h)

    def profile(self, enable: bool = True):
        _check(lib().rt3d_session_profile(self.h, int(enable)))

    PHASES = {1: "init_peaks", 2: "init_scan", 3: "init_spawn", 4: "grad_t", 5: "cand_t",
              6: "apss", 7: "grad_r", 8: "cand_r", 9: "knn", 10: "prune_a", 11: "prune_b",
              12: "grad_b", 13: "cand_b", 14: "fft", 15: "launch", 16: "apss_fit"}

    def profile_phases(self):
        """(name, duration_ns) per barrier-delimited phase of the last launch."""
        cap = 1 << 16
        buf = np.zeros(2 * cap, np.uint64)
        n = C.c_uint32()
        _check(lib().rt3d_profile_copy(self.h, ptr(buf, _u64), cap, C.byref(n)))
        r = Report()
        _check(lib().rt3d_report_info(self.h, C.byref(r)))
        pairs = buf[: 2 * n.value].reshape(-1, 2)
        out = []
        prev = None
        for pid, ts in pairs:
            out.append((self.PHASES.get(int(pid), str(pid)), 0 if prev is None else int(ts) - prev))
            prev = int(ts)
        return out

    KERNEL_CLASSES = ("stage_first", "stage_depth", "apss", "stage_intensity", "knn", "stage_tail",
                      "apss_fit", "iteration")

    def time_kernels(self, enable: bool = True):
        """CUDA events around every launch on the session stream (resets totals)."""
        _check(lib().rt3d_session_time_kernels(self.h, int(enable)))

    def graph_counts(self):
        """(graphs captured, graph launches) of this session so far."""
        c, n = _u64(), _u64()
        _check(lib().rt3d_graph_counts(self.h, C.byref(c), C.byref(n)))
        return c.value, n.value

    def kernel_times(self) -> dict:
        """{class: (total_ms, launches)} since time_kernels(); synchronizes."""
        ms = np.zeros(len(self.KERNEL_CLASSES))
        n = np.zeros(len(self.KERNEL_CLASSES), np.uint64)
        _check(lib().rt3d_kernel_times(self.h, ptr(ms, _dbl), ptr(n, _u64)))
        return {k: (float(ms[i]), int(n[i])) for i, k in enumerate(self.KERNEL_CLASSES)}

    def synchronize(self):
        _check(lib().rt3d_session_synchronize(self.h))

    def measure_fp64_peak(self) -> float:
        """Measured FP64 vector throughput of the device, TFLOP/s."""
        v = _dbl()
        _check(lib().rt3d_measure_fp64_peak(self.h, C.byref(v)))
        return v.value

    def after(self, prior: "Session"):
        """rt3d_session_after: this session's next work starts after the work
        queued so far on prior's stream (device-side, no host wait)."""
        _check(lib().rt3d_session_after(self.h, prior.h))

    def set_sharing(self, n_sessions: int):
        """Size the cooperative grids so n sessions can run frames concurrently."""
        _check(lib().rt3d_session_set_sharing(self.h, int(n_sessions)))

    def report(self) -> dict:
        r = Report()
        _check(lib().rt3d_report_info(self.h, C.byref(r)))
        it = r.iterations
        trace = np.zeros(it + 1)
        steps = np.zeros(max(it, 1), STEP_DIAG_DTYPE)
        _check(lib().rt3d_report_copy(self.h, ptr(trace, _dbl),
                                      steps.ctypes.data_as(P(StepDiag))))
        return dict(iterations=it, points=r.points, init_nll=r.init_nll, final_nll=r.final_nll,
                    init_seconds=r.init_seconds, iterate_seconds=r.iterate_seconds,
                    total_seconds=r.total_seconds, trace=trace, steps=steps[:it])

    def state(self):
        n = _u64()
        _check(lib().rt3d_state_size(self.h, C.byref(n)))
        pts = np.zeros(max(n.value, 1), POINT_DTYPE)
        bg = np.zeros(self.scene.n_pixels)
        _check(lib().rt3d_state_copy(self.h, ptr(pts, Point), ptr(bg, _dbl)))
        return pts[: n.value].copy(), bg

    # -- pipelined frames (rt3d_frame_submit / rt3d_frame_collect) ----------
    def frame_submit(self, sc: Scene, cfg: Config) -> int:
        """Enqueue H2D of sc's cube and its reconstruction; returns a ticket.
        sc's arrays must stay alive until the frame is collected."""
        cube, cfg_c = sc.cube_c(), cfg.to_c()
        t = _u64()
        _check(lib().rt3d_frame_submit(self.h, C.byref(cube), C.byref(cfg_c), C.byref(t)))
        if not hasattr(self, "_inflight"):
            self._inflight = {}
        self._inflight[t.value] = (sc, cube, cfg_c)
        return t.value

    def frame_collect(self, ticket: int, points: np.ndarray = None, background: np.ndarray = None):
        """Wait for a submitted frame; fills (or allocates) points / background.
        Returns (points[:n], background, report dict)."""
        sc, _, cfg_c = self._inflight[ticket]
        if points is None:
            cap = cfg_c.init.max_returns * sc.superres * sc.superres * sc.n_pixels
            points = np.zeros(max(cap, 1), POINT_DTYPE)
        if background is None:
            background = np.zeros(sc.n_pixels)
        n = _u64()
        r = Report()
        try:
            _check(lib().rt3d_frame_collect(self.h, ticket, ptr(points, Point), len(points),
                                            C.byref(n), ptr(background, _dbl), C.byref(r)))
        except Rt3dError as e:
            if e.status != 3:  # OUT_OF_RANGE: the frame stays in flight (collect again)
                self._inflight.pop(ticket, None)
            raise
        self._inflight.pop(ticket, None)
        rep = {"iterations": r.iterations, "points": int(r.points), "init_nll": r.init_nll,
               "final_nll": r.final_nll, "total_seconds": r.total_seconds}
        return points[: n.value], background, rep

    def reconstruct(self, cfg: Config) -> dict:
        self.reconstruct_async(cfg)
        rep = self.report()
        rep["points"], rep["background"] = self.state()
        return rep

    # -- operators -------------------------------------------------------
    def init_matched_filter(self, cfg: Config):
        ip = cfg.init_c()
        _check(lib().rt3d_init_matched_filter(self.h, C.byref(ip)))
        return self.state()

    def baseline_xcorr(self):
        _check(lib().rt3d_baseline_xcorr(self.h))
        return self.state()[0]

    def nll(self) -> float:
        v = _dbl()
        _check(lib().rt3d_nll(self.h, C.byref(v)))
        return v.value

    def grads(self) -> dict:
        n = len(self._keep[0])
        npix = self.scene.n_pixels
        out = {k: np.zeros(max(n, 1)) for k in ("gd", "gr", "cd", "cr")}
        out["oog"] = np.zeros(max(n, 1), np.uint8)
        out["gb"] = np.zeros(npix)
        out["cb"] = np.zeros(npix)
        L = lib()
        _check(L.rt3d_grad_depth(self.h, ptr(out["gd"], _dbl), ptr(out["oog"], _u8)))
        _check(L.rt3d_grad_intensity(self.h, ptr(out["gr"], _dbl)))
        _check(L.rt3d_grad_background(self.h, ptr(out["gb"], _dbl)))
        _check(L.rt3d_block_curvatures(self.h, ptr(out["cd"], _dbl), ptr(out["cr"], _dbl),
                                       ptr(out["cb"], _dbl)))
        for k in ("gd", "gr", "cd", "cr", "oog"):
            out[k] = out[k][:n]
        return out

    def palm_step(self, cfg: Config):
        c = cfg.to_c()
        d = StepDiag()
        _check(lib().rt3d_palm_step(self.h, C.byref(c), C.byref(d)))
        pts, bg = self.state()
        return pts, bg, d

    def matched_filter_peaks(self, events, irf_samples, tau_min, dtau, n_bins, k, thr, min_sep):
        from .abi import EVENT_DTYPE
        events = np.ascontiguousarray(events, EVENT_DTYPE)
        samples = np.ascontiguousarray(irf_samples, np.float64)
        f = Irf()
        f.tau_min, f.dtau = tau_min, dtau
        f.samples = ptr(samples, _dbl)
        f.n_samples = len(samples)
        out = np.zeros(max(k, 1), PEAK_DTYPE)
        n = _i32()
        _check(lib().rt3d_matched_filter_peaks(
            self.h, ptr(events, Event) if len(events) else None, len(events), C.byref(f), n_bins,
            k, thr, min_sep, out.ctypes.data_as(P(Peak)), C.byref(n)))
        return out[: n.value].copy()

    def apss_project(self, points, radius, min_nbrs=6, eps=1e-3, cell=None, index=None):
        points = np.ascontiguousarray(points, POINT_DTYPE)
        index = points if index is None else np.ascontiguousarray(index, POINT_DTYPE)
        out = np.zeros(len(points), POINT_DTYPE)
        ap = ApssParams()
        ap.kernel_radius, ap.min_neighbors, ap.sphere_degeneracy_eps = radius, min_nbrs, eps
        _check(lib().rt3d_apss_project(self.h, ptr(points, Point), len(points), C.byref(ap),
                                       ptr(index, Point), len(index),
                                       radius if cell is None else cell, ptr(out, Point)))
        return out

    def knn_filter(self, points, k, radius, cell=None, index=None):
        points = np.ascontiguousarray(points, POINT_DTYPE)
        index = points if index is None else np.ascontiguousarray(index, POINT_DTYPE)
        out = np.zeros(len(points), POINT_DTYPE)
        _check(lib().rt3d_knn_intensity_filter(self.h, ptr(points, Point), len(points), k,
                                               ptr(index, Point), len(index),
                                               radius if cell is None else cell, radius,
                                               ptr(out, Point)))
        return out

    def evaluate(self, est, truth, tau: float, pitch: float) -> dict:
        """evaluate (eval.hpp:33-87): recall / false-point rate / depth RMSE /
        intensity MAE of `est` against `truth`, matched per column of `pitch`."""
        est = np.ascontiguousarray(est, POINT_DTYPE)
        truth = np.ascontiguousarray(truth, POINT_DTYPE)
        e = Eval()
        _check(lib().rt3d_evaluate(self.h, ptr(est, Point), len(est), ptr(truth, Point),
                                   len(truth), tau, pitch, C.byref(e)))
        return {k: getattr(e, k) for k, _ in Eval._fields_}

    def simulate_cube(self, truth, background, seed: int):
        """simulate_cube's sampling (simulate.hpp:181-205) on the device into
        the session cube (sensor must be set).  Returns (n_events, signal
        photons, background photons)."""
        truth = np.ascontiguousarray(truth, POINT_DTYPE)
        bg = np.ascontiguousarray(background, np.float64)
        n = _u64()
        ph = (_u64 * 2)()
        _check(lib().rt3d_simulate_cube(self.h, ptr(truth, Point), len(truth), ptr(bg, _dbl),
                                        seed, C.byref(n), ph))
        return n.value, ph[0], ph[1]

    def cube_copy(self, npix: int, n_events: int):
        """The resident cube as (offsets u64[npix+1], events)."""
        off = np.zeros(npix + 1, np.uint64)
        ev = np.zeros(max(n_events, 1), EVENT_DTYPE)
        _check(lib().rt3d_cube_copy(self.h, ptr(off, _u64), ptr(ev, Event)))
        return off, ev[:n_events]

    def prune(self, points, r_min):
        points = np.ascontiguousarray(points, POINT_DTYPE)
        out = np.zeros(max(len(points), 1), POINT_DTYPE)
        n = _u64()
        _check(lib().rt3d_prune(self.h, ptr(points, Point), len(points), r_min, ptr(out, Point),
                                C.byref(n)))
        return out[: n.value].copy()

    def fft_lowpass(self, img, cutoff, clamp=False):
        img = np.ascontiguousarray(img, np.float64)
        out = np.zeros_like(img)
        _check(lib().rt3d_fft_lowpass_filter(self.h, ptr(img, _dbl), img.shape[0], img.shape[1],
                                             cutoff, int(clamp), ptr(out, _dbl)))
        return out
