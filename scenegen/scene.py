"""Synthetic scenes (scenegen/libscene.so, scenegen/rt3d_scene.h): a restatement of the
reference's simulate_cube (simulate.hpp:139-223) used to make benchmark
inputs of the shapes BASELINE.json names."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from pathlib import Path
from typing import List, Optional, Sequence, Tuple

import numpy as np

from paper_1905_06700_b200.abi import EVENT_DTYPE, POINT_DTYPE, Event, Point, Scene, ptr

LIB_PATH = Path(__file__).resolve().parent / "libscene.so"


class Surface(C.Structure):
    _fields_ = [
        ("kind", C.c_int32), ("checker_period", C.c_int32), ("depth_m", C.c_double),
        ("slope_x", C.c_double), ("slope_y", C.c_double), ("bump_amp", C.c_double),
        ("bump_cx", C.c_double), ("bump_cy", C.c_double), ("bump_width", C.c_double),
        ("reflectivity", C.c_double), ("checker_contrast", C.c_double),
        ("region", C.c_int32 * 4), ("n_holes", C.c_int32), ("pad_", C.c_int32),
        ("holes", C.POINTER(C.c_int32)),
    ]


class SpecC(C.Structure):
    _fields_ = [
        ("rows", C.c_int32), ("cols", C.c_int32), ("bins", C.c_int32), ("superres", C.c_int32),
        ("bin_resolution_m", C.c_double), ("pixel_pitch_m", C.c_double),
        ("irf_sigma_bins", C.c_double), ("irf_support_sigmas", C.c_double),
        ("ambient_per_bin", C.c_double), ("target_ppp", C.c_double), ("target_sbr", C.c_double),
        ("n_surfaces", C.c_int32), ("n_dead", C.c_int32), ("surfaces", C.POINTER(Surface)),
        ("dead_pixels", C.POINTER(C.c_int32)),
    ]


@dataclass
class SurfaceSpec:
    """SurfaceSpec (simulate.hpp:20-42)."""
    kind: str = "plane"
    depth_m: float = 0.0
    slope_x: float = 0.0
    slope_y: float = 0.0
    bump_amp: float = 0.0
    bump_cx: float = 0.0
    bump_cy: float = 0.0
    bump_width: float = 1.0
    reflectivity: float = 1.0
    checker_contrast: float = 0.0
    checker_period: int = 8
    region: Tuple[int, int, int, int] = (0, 0, -1, -1)
    holes: Sequence[Tuple[int, int, int, int]] = ()


@dataclass
class SceneSpec:
    """SceneSpec (simulate.hpp:47-65) with its defaults."""
    rows: int = 32
    cols: int = 32
    bins: int = 256
    superres: int = 1
    bin_resolution_m: float = 0.01
    pixel_pitch_m: float = 0.02
    irf_sigma_bins: float = 1.5
    irf_support_sigmas: float = 4.0
    ambient_per_bin: float = 0.0
    target_ppp: float = -1.0
    target_sbr: float = -1.0
    surfaces: List[SurfaceSpec] = field(default_factory=list)
    dead_pixels: Sequence[Tuple[int, int]] = ()


_lib: Optional[C.CDLL] = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(f"{LIB_PATH} missing: run __graft_entry__.build()")
        L = C.CDLL(str(LIB_PATH))
        L.rt3d_scene_simulate.restype = C.c_int
        L.rt3d_scene_simulate.argtypes = [C.POINTER(SpecC), C.c_uint64, C.c_int, C.POINTER(C.c_void_p)]
        L.rt3d_scene_error.restype = C.c_char_p
        L.rt3d_scene_sizes.argtypes = [C.c_void_p] + [C.POINTER(C.c_uint64)] * 3
        L.rt3d_scene_copy.argtypes = [C.c_void_p, C.POINTER(C.c_uint64), C.POINTER(Event),
                                      C.POINTER(C.c_double), C.POINTER(Point),
                                      C.POINTER(C.c_uint8), C.POINTER(C.c_double)]
        L.rt3d_scene_free.argtypes = [C.c_void_p]
        L.rt3d_scene_background.argtypes = [C.c_void_p, C.POINTER(C.c_double)]
        _lib = L
    return _lib


def simulate(spec: SceneSpec, seed: int, threads: int = 0) -> Scene:
    """simulate_cube(spec, build_sensor(spec), seed) -> Scene (+ .truth)."""
    keep = []
    surfs = (Surface * max(1, len(spec.surfaces)))()
    for k, s in enumerate(spec.surfaces):
        c = surfs[k]
        c.kind = 0 if s.kind == "plane" else 1
        c.checker_period = s.checker_period
        for f in ("depth_m", "slope_x", "slope_y", "bump_amp", "bump_cx", "bump_cy",
                  "bump_width", "reflectivity", "checker_contrast"):
            setattr(c, f, getattr(s, f))
        c.region[:] = list(s.region)
        holes = np.ascontiguousarray(np.array(s.holes, np.int32).reshape(-1))
        keep.append(holes)
        c.n_holes = len(s.holes)
        c.holes = ptr(holes, C.c_int32) if len(s.holes) else None
    dead = np.ascontiguousarray(np.array(spec.dead_pixels, np.int32).reshape(-1))
    sp = SpecC(spec.rows, spec.cols, spec.bins, spec.superres, spec.bin_resolution_m,
               spec.pixel_pitch_m, spec.irf_sigma_bins, spec.irf_support_sigmas,
               spec.ambient_per_bin, spec.target_ppp, spec.target_sbr, len(spec.surfaces),
               len(spec.dead_pixels), surfs, ptr(dead, C.c_int32) if len(dead) else None)
    L = lib()
    h = C.c_void_p()
    if L.rt3d_scene_simulate(C.byref(sp), seed, threads, C.byref(h)) != 0:
        raise ValueError(L.rt3d_scene_error().decode())
    ne, nt, ni = C.c_uint64(), C.c_uint64(), C.c_uint64()
    L.rt3d_scene_sizes(h, C.byref(ne), C.byref(nt), C.byref(ni))
    npix = spec.rows * spec.cols
    offsets = np.zeros(npix + 1, np.uint64)
    events = np.zeros(max(ne.value, 1), EVENT_DTYPE)
    irf = np.zeros(ni.value)
    truth = np.zeros(max(nt.value, 1), POINT_DTYPE)
    deadm = np.zeros(npix, np.uint8)
    meta = np.zeros(5)
    L.rt3d_scene_copy(h, ptr(offsets, C.c_uint64), events.ctypes.data_as(C.POINTER(Event)),
                      ptr(irf, C.c_double), truth.ctypes.data_as(C.POINTER(Point)),
                      ptr(deadm, C.c_uint8), ptr(meta, C.c_double))
    bg = np.zeros(npix)
    L.rt3d_scene_background(h, ptr(bg, C.c_double))
    L.rt3d_scene_free(h)
    sc = Scene(spec.rows, spec.cols, spec.bins, offsets, events[: ne.value], irf, meta[0],
               meta[1], superres=spec.superres, pixel_pitch=spec.pixel_pitch_m,
               bin_resolution=spec.bin_resolution_m, bin_width_s=meta[2], dead=deadm)
    sc.truth = truth[: nt.value].copy()
    sc.background_truth = bg
    sc.signal_photons, sc.background_photons = int(meta[3]), int(meta[4])
    return sc


def encode_spcb(sc) -> bytes:
    """encode_cube (io.hpp:99-114): 'SPCB', version 1, rows, cols, bins (u32
    little-endian), bin width (f64), then per pixel its event count and
    (bin, count) pairs."""
    import struct
    out = [b"SPCB", struct.pack("<4I", 1, sc.n_rows, sc.n_cols, sc.n_bins),
           struct.pack("<d", float(sc.bin_width_s))]
    off = np.asarray(sc.offsets, np.uint64)
    ev = np.ascontiguousarray(sc.events)
    counts = np.diff(off).astype(np.uint32)
    words = np.empty(len(counts) + 2 * len(ev), np.uint32)
    # record p at word (p + 2 off[p]): count, then its events
    pos = np.arange(len(counts), dtype=np.uint64) + 2 * off[:-1]
    words[pos.astype(np.int64)] = counts
    if len(ev):
        pix = np.repeat(np.arange(len(counts)), counts.astype(np.int64))
        k = np.arange(len(ev), dtype=np.uint64) - off[pix]
        w = (pos[pix] + 1 + 2 * k).astype(np.int64)
        words[w] = ev["bin"]
        words[w + 1] = ev["count"]
    out.append(words.astype("<u4").tobytes())
    return b"".join(out)
