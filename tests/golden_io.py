"""Load the committed golden fixtures (tests/golden/*.npz, made by
tests/golden/make_golden.py from the reference itself)."""
from __future__ import annotations

import ast
from functools import lru_cache
from pathlib import Path

import numpy as np

from paper_1905_06700_b200.abi import EVENT_DTYPE, Config, Scene

GOLDEN = Path(__file__).resolve().parent / "golden"
SCENE_NAMES = ["small_s3", "small_s13", "two_surface_24", "superres_8", "dense_12"]


def _scene(d, prefix="") -> Scene:
    g = lambda k: d[prefix + k]
    ev = np.ascontiguousarray(g("events"), np.uint32).view(EVENT_DTYPE).reshape(-1)
    sc = Scene(int(g("rows")), int(g("cols")), int(g("bins")), g("offsets"), ev, g("irf"),
               float(g("tau_min")), float(g("dtau")), superres=int(g("superres")),
               pixel_pitch=float(g("pitch")), bin_resolution=float(g("bres")),
               bin_width_s=float(g("bin_width_s")), gain=g("gain"), dead=g("dead"))
    if prefix + "points" in d:
        sc.with_state(g("points"), g("background"))
    return sc


@lru_cache(None)
def _load(name):
    return dict(np.load(GOLDEN / name, allow_pickle=False))


def random_seeds():
    return [int(s) for s in _load("random_instances.npz")["seeds"]]


def random_instance(seed):
    d = _load("random_instances.npz")
    sc = _scene(d, f"r{seed}_")
    exp = {k[len(f"r{seed}_"):]: d[k] for k in d if k.startswith(f"r{seed}_")}
    return sc, exp


def scene(name):
    d = _load(f"scene_{name}.npz")
    sc = _scene(d)
    cfg = Config(**ast.literal_eval(str(d["cfg"])))
    return sc, cfg, d


def peaks():
    return _load("peaks.npz")


def denoise():
    return _load("denoise.npz")
