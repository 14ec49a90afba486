"""ctypes mirror of include/rt3d.h plus numpy dtypes for the C views.

Plain data plumbing: the structs below must match include/rt3d.h byte for
byte (tests/test_abi.py checks sizes and offsets against the compiled
library).  Host-side data is kept in numpy arrays; `Scene` bundles a cube, a
sensor and optionally a state and hands out ctypes views that point into the
numpy buffers (no copies).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

# ---- numpy dtypes ---------------------------------------------------------
EVENT_DTYPE = np.dtype([("bin", "<u4"), ("count", "<u4")])
POINT_DTYPE = np.dtype(
    [
        ("x", "<f8"), ("y", "<f8"), ("z", "<f8"), ("intensity", "<f8"),
        ("i", "<i4"), ("j", "<i4"), ("fi", "<i4"), ("fj", "<i4"),
        ("t", "<f8"), ("flags", "u1"), ("pad", "u1", (7,)),
    ]
)
assert POINT_DTYPE.itemsize == 64
PEAK_DTYPE = np.dtype([("t", "<f8"), ("response", "<f8"), ("mass", "<f8")])

FLAG_ISOLATED, FLAG_OUT_OF_GATE, FLAG_DEGENERATE = 1, 2, 4

STATUS = {
    0: "OK", 1: "INVALID_ARGUMENT", 2: "FORMAT", 3: "OUT_OF_RANGE", 4: "CUDA",
    5: "NCCL", 6: "UNSUPPORTED", 7: "NO_DEVICE",
}


# ---- ctypes structs -------------------------------------------------------
class Event(C.Structure):
    _fields_ = [("bin", C.c_uint32), ("count", C.c_uint32)]


class Point(C.Structure):
    _fields_ = [
        ("x", C.c_double), ("y", C.c_double), ("z", C.c_double), ("intensity", C.c_double),
        ("i", C.c_int32), ("j", C.c_int32), ("fi", C.c_int32), ("fj", C.c_int32),
        ("t", C.c_double), ("flags", C.c_uint8), ("pad_", C.c_uint8 * 7),
    ]


class Irf(C.Structure):
    _fields_ = [
        ("tau_min", C.c_double), ("dtau", C.c_double),
        ("samples", C.POINTER(C.c_double)), ("n_samples", C.c_uint64),
    ]


class Sensor(C.Structure):
    _fields_ = [
        ("n_rows", C.c_int32), ("n_cols", C.c_int32), ("n_bins", C.c_int32),
        ("superres", C.c_int32), ("pixel_pitch", C.c_double), ("bin_resolution", C.c_double),
        ("irf_shared", Irf), ("irf_per_pixel", C.POINTER(Irf)),
        ("gain", C.POINTER(C.c_double)), ("dead", C.POINTER(C.c_uint8)),
    ]


class Cube(C.Structure):
    _fields_ = [
        ("n_rows", C.c_int32), ("n_cols", C.c_int32), ("n_bins", C.c_int32), ("pad_", C.c_int32),
        ("bin_width_s", C.c_double), ("offsets", C.POINTER(C.c_uint64)),
        ("events", C.POINTER(Event)), ("n_events", C.c_uint64),
    ]


class StateView(C.Structure):
    _fields_ = [
        ("points", C.POINTER(Point)), ("n_points", C.c_uint64),
        ("background", C.POINTER(C.c_double)), ("bucket_offsets", C.POINTER(C.c_uint32)),
        ("bucket_points", C.POINTER(C.c_uint32)),
    ]


class InitParams(C.Structure):
    _fields_ = [("max_returns", C.c_int32), ("min_separation", C.c_int32),
                ("peak_threshold", C.c_double)]


class ApssParams(C.Structure):
    _fields_ = [("kernel_radius", C.c_double), ("sphere_degeneracy_eps", C.c_double),
                ("min_neighbors", C.c_int32), ("pad_", C.c_int32)]


class ReconConfig(C.Structure):
    _fields_ = [
        ("max_iters", C.c_int32), ("knn_k", C.c_int32), ("stop_tol", C.c_double),
        ("step_t_auto", C.c_int32), ("step_r_auto", C.c_int32), ("step_b_auto", C.c_int32),
        ("background_mode", C.c_int32),
        ("step_t", C.c_double), ("step_r", C.c_double), ("step_b", C.c_double),
        ("backtrack_beta", C.c_double), ("apss", ApssParams), ("r_min", C.c_double),
        ("fft_cutoff", C.c_double), ("init", InitParams),
    ]


class Peak(C.Structure):
    _fields_ = [("t", C.c_double), ("response", C.c_double), ("mass", C.c_double)]


class BlockDiag(C.Structure):
    _fields_ = [("step_used", C.c_double), ("nll_after_grad", C.c_double),
                ("nll_after_denoise", C.c_double), ("backtracks", C.c_int32), ("pad_", C.c_int32)]


class StepDiag(C.Structure):
    _fields_ = [
        ("nll_before", C.c_double), ("nll_after", C.c_double),
        ("points_before", C.c_uint64), ("points_after", C.c_uint64),
        ("depth", BlockDiag), ("intensity", BlockDiag), ("background", BlockDiag),
    ]


class Report(C.Structure):
    _fields_ = [
        ("iterations", C.c_int32), ("pad_", C.c_int32), ("points", C.c_uint64),
        ("init_nll", C.c_double), ("final_nll", C.c_double), ("init_seconds", C.c_double),
        ("iterate_seconds", C.c_double), ("total_seconds", C.c_double),
    ]


STEP_DIAG_DTYPE = np.dtype(
    [
        ("nll_before", "<f8"), ("nll_after", "<f8"), ("points_before", "<u8"),
        ("points_after", "<u8"),
    ]
    + [
        (f"{b}_{f}", t)
        for b in ("depth", "intensity", "background")
        for f, t in (("step_used", "<f8"), ("nll_after_grad", "<f8"),
                     ("nll_after_denoise", "<f8"), ("backtracks", "<i4"), ("pad", "<i4"))
    ]
)
assert STEP_DIAG_DTYPE.itemsize == C.sizeof(StepDiag)


def ptr(a: np.ndarray, ctype):
    """Pointer into a C-contiguous numpy buffer."""
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(C.POINTER(ctype))


# ---- configs --------------------------------------------------------------
@dataclass
class Config:
    """splidar::ReconConfig (reconstruct.hpp:56-66) with its defaults."""
    max_iters: int = 50
    stop_tol: float = 1e-4
    step_t: Optional[float] = None  # None = "auto"
    step_r: Optional[float] = None
    step_b: Optional[float] = None
    backtrack_beta: float = 0.5
    apss_radius: float = 0.1
    apss_min_neighbors: int = 6
    apss_degeneracy_eps: float = 1e-3
    knn_k: int = 9
    r_min: float = 0.0
    background_mode: int = 0
    fft_cutoff: float = 0.5
    init_max_returns: int = 3
    init_peak_threshold: float = 0.5
    init_min_separation: int = 3

    def to_c(self) -> ReconConfig:
        c = ReconConfig()
        c.max_iters = self.max_iters
        c.knn_k = self.knn_k
        c.stop_tol = self.stop_tol
        c.step_t_auto = int(self.step_t is None)
        c.step_r_auto = int(self.step_r is None)
        c.step_b_auto = int(self.step_b is None)
        c.step_t = 1.0 if self.step_t is None else self.step_t
        c.step_r = 1.0 if self.step_r is None else self.step_r
        c.step_b = 1.0 if self.step_b is None else self.step_b
        c.backtrack_beta = self.backtrack_beta
        c.background_mode = self.background_mode
        c.apss.kernel_radius = self.apss_radius
        c.apss.min_neighbors = self.apss_min_neighbors
        c.apss.sphere_degeneracy_eps = self.apss_degeneracy_eps
        c.r_min = self.r_min
        c.fft_cutoff = self.fft_cutoff
        c.init.max_returns = self.init_max_returns
        c.init.peak_threshold = self.init_peak_threshold
        c.init.min_separation = self.init_min_separation
        return c

    def init_c(self) -> InitParams:
        return self.to_c().init

    def apss_c(self) -> ApssParams:
        return self.to_c().apss


# ---- scene bundle ---------------------------------------------------------
@dataclass
class Scene:
    """Cube + sensor (+ optional state) as numpy arrays, with ctypes views."""
    n_rows: int
    n_cols: int
    n_bins: int
    offsets: np.ndarray           # u64[npix+1]
    events: np.ndarray            # EVENT_DTYPE[E]
    irf_samples: np.ndarray       # f8, normalised
    irf_tau_min: float
    irf_dtau: float
    superres: int = 1
    pixel_pitch: float = 1.0
    bin_resolution: float = 1.0
    bin_width_s: float = 1e-9
    gain: Optional[np.ndarray] = None
    dead: Optional[np.ndarray] = None
    points: Optional[np.ndarray] = None      # POINT_DTYPE
    background: Optional[np.ndarray] = None  # f8[npix]
    # SensorModel::irf_per_pixel (sensor.hpp:160-164): None, or npix
    # (samples, tau_min, dtau) tuples in row-major pixel order
    irf_per_pixel: Optional[list] = None
    _keep: list = field(default_factory=list, repr=False)

    def __post_init__(self):
        npix = self.n_rows * self.n_cols
        self.offsets = np.ascontiguousarray(self.offsets, dtype=np.uint64)
        self.events = np.ascontiguousarray(self.events, dtype=EVENT_DTYPE)
        self.irf_samples = np.ascontiguousarray(self.irf_samples, dtype=np.float64)
        if self.gain is None:
            self.gain = np.ones(npix)
        if self.dead is None:
            self.dead = np.zeros(npix, np.uint8)
        self.gain = np.ascontiguousarray(self.gain, dtype=np.float64)
        self.dead = np.ascontiguousarray(self.dead, dtype=np.uint8)

    @property
    def n_pixels(self) -> int:
        return self.n_rows * self.n_cols

    def cube_c(self) -> Cube:
        c = Cube()
        c.n_rows, c.n_cols, c.n_bins = self.n_rows, self.n_cols, self.n_bins
        c.bin_width_s = self.bin_width_s
        c.offsets = ptr(self.offsets, C.c_uint64)
        c.events = ptr(self.events, Event)
        c.n_events = len(self.events)
        return c

    def irf_c(self) -> Irf:
        f = Irf()
        f.tau_min = self.irf_tau_min
        f.dtau = self.irf_dtau
        f.samples = ptr(self.irf_samples, C.c_double)
        f.n_samples = len(self.irf_samples)
        return f

    def sensor_c(self) -> Sensor:
        s = Sensor()
        s.n_rows, s.n_cols, s.n_bins = self.n_rows, self.n_cols, self.n_bins
        s.superres = self.superres
        s.pixel_pitch = self.pixel_pitch
        s.bin_resolution = self.bin_resolution
        s.irf_shared = self.irf_c()
        s.irf_per_pixel = None
        if self.irf_per_pixel is not None:
            assert len(self.irf_per_pixel) == self.n_pixels
            arr = (Irf * self.n_pixels)()
            keep = []
            for k, (smp, tmin, dt) in enumerate(self.irf_per_pixel):
                smp = np.ascontiguousarray(smp, np.float64)
                keep.append(smp)
                arr[k].tau_min, arr[k].dtau = float(tmin), float(dt)
                arr[k].samples = ptr(smp, C.c_double)
                arr[k].n_samples = len(smp)
            self._keep = [arr, keep]
            s.irf_per_pixel = C.cast(arr, C.POINTER(Irf))
        s.gain = ptr(self.gain, C.c_double)
        s.dead = ptr(self.dead, C.c_uint8)
        return s

    def with_state(self, points: np.ndarray, background: np.ndarray) -> "Scene":
        self.points = np.ascontiguousarray(points, dtype=POINT_DTYPE)
        self.background = np.ascontiguousarray(background, dtype=np.float64)
        return self


def buckets(points: np.ndarray, n_rows: int, n_cols: int):
    """SceneState::refresh (likelihood.hpp:38-55): stable counting sort."""
    pix = points["i"].astype(np.int64) * n_cols + points["j"].astype(np.int64)
    counts = np.bincount(pix, minlength=n_rows * n_cols).astype(np.uint32)
    offsets = np.zeros(n_rows * n_cols + 1, np.uint32)
    np.cumsum(counts, out=offsets[1:])
    order = np.argsort(pix, kind="stable").astype(np.uint32)
    return offsets, order
