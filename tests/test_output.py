"""Output formats after the path: rt3d_encode_ply
against the reference's encode_ply (io.hpp:162-179, through oracle/_ref) and
a restatement; rt3d_encode_background_csv against the CLI's writer
(tools/splidar_main.cpp:204-212), restated here.  Host-only formatting: no
device needed."""
import ctypes as C

import numpy as np
import pytest

import golden_io as G
import oracle_lib as O
from paper_1905_06700_b200 import rt3d
from paper_1905_06700_b200.abi import POINT_DTYPE, Point, ptr


def _cloud(n, seed):
    rng = np.random.default_rng(seed)
    p = np.zeros(n, POINT_DTYPE)
    p["x"] = rng.uniform(0, 3, n)
    p["y"] = rng.uniform(-1, 1, n) * 10.0 ** rng.integers(-9, 9, n)
    p["z"] = rng.uniform(0, 50, n)
    p["intensity"] = rng.exponential(1.0, n)
    p["intensity"][::7] = 0.0
    if n > 3:
        p["x"][1] = -0.0
        p["y"][2] = 123456789.5
        p["z"][3] = 1e-310          # subnormal
    return p


def _restated_ply(p, pitch=None):
    """io.hpp:162-179 restated with Python's (correctly rounded) %-format."""
    out = ["ply\nformat ascii 1.0\n"]
    if pitch is not None:
        out.append("comment pixel_pitch %.17g\n" % pitch)
    out.append("element vertex %d\n" % len(p))
    out.append("property float x\nproperty float y\nproperty float z\n"
               "property float intensity\nend_header\n")
    for q in p:
        out.append("%.9g %.9g %.9g %.9g\n" % (q["x"], q["y"], q["z"], q["intensity"]))
    return "".join(out).encode()


_REF_PLY_CHILD = r"""
import ctypes as C, sys
lib = C.CDLL(sys.argv[1])
data = sys.stdin.buffer.read()
n, has, pitch = len(data) // 64, int(sys.argv[2]), float(sys.argv[3])
pts = C.create_string_buffer(data, max(len(data), 1))
nb = C.c_uint64()
args = (pts, C.c_uint64(n), has, C.c_double(pitch))
assert lib.ref_encode_ply(*args, None, C.c_uint64(0), C.byref(nb)) == 0
out = C.create_string_buffer(max(nb.value, 1))
assert lib.ref_encode_ply(*args, out, nb, C.byref(nb)) == 0
sys.stdout.buffer.write(out.raw[: nb.value])
"""


def _ref_ply(p, pitch=None):
    """The reference's encode_ply through oracle/_ref, in a child process:
    libref.so carries its own static libstdc++, whose iostreams must not share
    a process with the libstdc++ numpy loads."""
    import subprocess
    import sys
    r = subprocess.run([sys.executable, "-c", _REF_PLY_CHILD, str(O.REF_SO),
                        str(int(pitch is not None)), repr(float(pitch or 0.0))],
                       input=np.ascontiguousarray(p, POINT_DTYPE).tobytes(),
                       capture_output=True, check=True)
    return r.stdout


@pytest.mark.parametrize("n,pitch", [(0, None), (1, 0.02), (257, None), (40000, 0.0025)])
def test_ply_matches_restatement(n, pitch):
    p = _cloud(n, n + 1)
    assert rt3d.encode_ply(p, pitch) == _restated_ply(p, pitch)


@pytest.mark.parametrize("n,pitch", [(0, 0.02), (300, None), (70000, 0.05)])
def test_ply_matches_reference(n, pitch):
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    p = _cloud(n, 7 * n + 3)
    assert rt3d.encode_ply(p, pitch) == _ref_ply(p, pitch)


def test_ply_of_golden_cloud_matches_reference():
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    _, _, d = G.scene("superres_8")
    pts = np.ascontiguousarray(d["rec_points"]).view(POINT_DTYPE).reshape(-1)
    assert len(pts) > 0
    assert rt3d.encode_ply(pts, float(d["pitch"])) == _ref_ply(pts, float(d["pitch"]))
    bg = np.asarray(d["rec_background"], np.float64).reshape(int(d["rows"]), int(d["cols"]))
    assert rt3d.encode_background_csv(bg) == _restated_csv(bg)


def _restated_csv(bg):
    rows, cols = bg.shape
    return "".join("%.9g" % bg[i, j] + ("\n" if j + 1 == cols else ",")
                   for i in range(rows) for j in range(cols)).encode()


@pytest.mark.parametrize("rows,cols", [(0, 0), (1, 1), (3, 5), (141, 141), (300, 257)])
def test_background_csv(rows, cols):
    rng = np.random.default_rng(rows * 1000 + cols)
    bg = rng.exponential(1e-3, (rows, cols))
    if bg.size:
        bg.flat[0] = 1e-6
    assert rt3d.encode_background_csv(bg) == _restated_csv(bg)


def test_bad_arguments():
    n = C.c_uint64()
    L = rt3d.lib()
    assert L.rt3d_encode_ply(None, 5, 0, 0.0, None, 0, C.byref(n)) == 1
    assert L.rt3d_encode_background_csv(None, -1, 2, None, 0, C.byref(n)) == 1
