"""The SURVEY.md §8d benchmark workloads (BASELINE.json configs A-E) as
SceneSpecs + ReconConfigs, shared by bench.py, the parity tests and tools.

`spec_text()` renders a SceneSpec as the reference's key=value scene file
(SceneSpec::from_kv, simulate.hpp:225-302), so the reference arm and the
parity tests can build the same cube with the reference's own simulate_cube
(oracle/_ref/libref.so, `oracle_lib.ref_simulate`).
"""
from __future__ import annotations

import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

from paper_1905_06700_b200.abi import Config  # noqa: E402
from scenegen.scene import SceneSpec, SurfaceSpec  # noqa: E402


def acceptance_cfg(**kw) -> Config:
    """The acceptance preset (acceptance_main.cpp:70-80) with a fixed budget
    (bench_scaling, eval.hpp:216-217: stop_tol 0)."""
    base = dict(max_iters=25, stop_tol=0.0, apss_radius=0.16, knn_k=9, r_min=0.25,
                init_max_returns=3, init_peak_threshold=0.5, init_min_separation=6)
    base.update(kw)
    return Config(**base)


def config_a():
    spec = SceneSpec(rows=64, cols=64, bins=1024, bin_resolution_m=0.01, pixel_pitch_m=0.02,
                     irf_sigma_bins=1.5, target_ppp=50.0, target_sbr=1.0,
                     surfaces=[SurfaceSpec(depth_m=7.0),
                               SurfaceSpec(depth_m=5.0, region=(16, 16, 48, 48))])
    return "A 64x64x1024 two planes, ~100 photons/px", spec, 100, acceptance_cfg()


def config_b():
    """141x141 px, 4613 bins of 0.3 mm, 3 ppp, SBR 13."""
    pitch = 0.0025
    spec = SceneSpec(
        rows=141, cols=141, bins=4613, bin_resolution_m=0.0003, pixel_pitch_m=pitch,
        irf_sigma_bins=1.5, target_ppp=3.0, target_sbr=13.0,
        surfaces=[
            SurfaceSpec(depth_m=1.2, holes=[(40, 30, 101, 121)]),
            SurfaceSpec(kind="bump", depth_m=1.0, bump_amp=-0.12, bump_width=0.06,
                        bump_cx=70.5 * pitch, bump_cy=75.5 * pitch, region=(35, 25, 106, 126)),
        ])
    return ("141x141 px x 4613 bins polystyrene-head-like synthetic frame", spec, 141,
            acceptance_cfg(apss_radius=0.02))


def config_c(frame: int = 0):
    """32x32 px, 153 bins, superres 3, ~900 photons/px; the
    person bump moves one fine pixel per frame."""
    s, pitch = 3, 0.05
    spec = SceneSpec(rows=32, cols=32, bins=153, superres=s, bin_resolution_m=0.0375,
                     pixel_pitch_m=pitch, irf_sigma_bins=1.5, target_ppp=450.0, target_sbr=1.0,
                     surfaces=[
                         SurfaceSpec(depth_m=1.5, holes=[(10, 10, 20, 20), (40, 50, 55, 70),
                                                         (70, 20, 85, 35)]),
                         SurfaceSpec(kind="bump", depth_m=3.0, bump_amp=-0.2, bump_width=0.4,
                                     bump_cx=(30 + frame) * pitch, bump_cy=48 * pitch,
                                     region=(10, 20, 80, 76)),
                         SurfaceSpec(depth_m=4.5)])
    return ("C 32x32x153 superres 3 (96x96), three surfaces, ~900 photons/px", spec,
            1000 + frame, acceptance_cfg(apss_radius=0.30, r_min=0.2))


def _camouflage(n, scale):
    """Configs D / E: a camouflage net with a grid of holes at 5 m, a target
    bump at 8 m, a back plane at 12 m (<= 3 surfaces per px)."""
    pitch = 0.02
    step, hole = 16 * scale, 8 * scale
    holes = [(a, b, a + hole, b + hole) for a in range(0, n, step) for b in range(0, n, step)]
    c = n * pitch / 2
    return [SurfaceSpec(depth_m=5.0, holes=holes),
            SurfaceSpec(kind="bump", depth_m=8.0, bump_amp=-0.5, bump_cx=c, bump_cy=c,
                        bump_width=0.4 * c),
            SurfaceSpec(depth_m=12.0)]


def config_d():
    spec = SceneSpec(rows=256, cols=256, bins=2048, bin_resolution_m=0.01, pixel_pitch_m=0.02,
                     irf_sigma_bins=1.5, target_ppp=30.0, target_sbr=1.0,
                     surfaces=_camouflage(256, 1))
    return "D 256x256x2048 camouflage, ~60 photons/px", spec, 256, acceptance_cfg()


def config_e():
    spec = SceneSpec(rows=1024, cols=1024, bins=2048, bin_resolution_m=0.01, pixel_pitch_m=0.02,
                     irf_sigma_bins=1.5, target_ppp=50.0, target_sbr=1.0,
                     surfaces=_camouflage(1024, 4))
    return "E 1024x1024x2048 camouflage, ~100 photons/px", spec, 1024, acceptance_cfg()


CONFIGS = {"A": config_a, "B": config_b, "C": config_c, "D": config_d, "E": config_e}


def _num(v) -> str:
    return repr(float(v)) if isinstance(v, float) else str(v)


def spec_text(spec: SceneSpec) -> str:
    """SceneSpec -> the reference's scene file text (simulate.hpp:225-302).
    Doubles use Python's shortest round-trip repr, which strtod reads back to
    the same bits."""
    lines = [f"{k} = {_num(getattr(spec, k))}" for k in (
        "rows", "cols", "bins", "superres", "bin_resolution_m", "pixel_pitch_m",
        "irf_sigma_bins", "irf_support_sigmas", "ambient_per_bin", "target_ppp", "target_sbr")]
    if spec.dead_pixels:
        lines.append("dead_pixels = " + "; ".join(f"{i},{j}" for i, j in spec.dead_pixels))
    for s in spec.surfaces:
        lines.append("[surface]")
        lines.append(f"type = {s.kind}")
        for k in ("depth_m", "slope_x", "slope_y", "bump_amp", "bump_cx", "bump_cy",
                  "bump_width", "reflectivity", "checker_contrast"):
            lines.append(f"{k} = {_num(float(getattr(s, k)))}")
        lines.append(f"checker_period = {int(s.checker_period)}")
        if tuple(s.region) != (0, 0, -1, -1):
            lines.append("region = " + ",".join(str(int(v)) for v in s.region))
        if s.holes:
            lines.append("holes = " + "; ".join(",".join(str(int(v)) for v in h) for h in s.holes))
    return "\n".join(lines) + "\n"
