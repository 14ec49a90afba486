"""SPCB ingest (io.hpp:99-145): the Python encoder against the reference's
encode_cube / decode_cube (CPU, where the reference library is built), and
the device decode (rt3d_set_cube_spcb) against the host CSR path (GPU)."""
import ctypes as C
import struct

import numpy as np
import pytest

import golden_io as G
import oracle_lib as O
from scenegen.scene import encode_spcb


def _ref_encode(sc):
    lib = O.ref()
    lib.ref_encode_cube.restype = C.c_int
    n = C.c_uint64()
    cube = sc.cube_c()
    assert lib.ref_encode_cube(C.byref(cube), None, 0, C.byref(n)) == 0
    out = np.zeros(n.value, np.uint8)
    assert lib.ref_encode_cube(C.byref(cube), out.ctypes.data_as(C.POINTER(C.c_uint8)), n.value,
                               C.byref(n)) == 0
    return out.tobytes()


def _ref_decode_error(data: bytes):
    lib = O.ref()
    buf = np.frombuffer(data, np.uint8).copy()
    rc = lib.ref_decode_cube(buf.ctypes.data_as(C.POINTER(C.c_uint8)), len(buf), None, None, 0)
    return None if rc == 0 else lib.ref_last_error().decode()


def _bad_cases(sc):
    good = encode_spcb(sc)
    w = np.frombuffer(good[28:], "<u4").copy()
    cases = {
        "magic": b"SPCX" + good[4:],
        "version": good[:4] + struct.pack("<I", 2) + good[8:],
        "zero": good[:8] + struct.pack("<I", 0) + good[12:],
        "trailing": good + b"\0",
        "truncated_bin": good[:-8],
        "truncated_value": good[:-4],
        "truncated_header": good[:20],
    }
    # first event of the first nonempty pixel: bin out of range / zero count
    p = int(np.argmax(np.diff(sc.offsets) > 0))
    e0 = int(sc.offsets[p])
    w0 = p + 1 + 2 * e0  # word of that event's bin (after the count word)
    a = w.copy()
    a[w0] = sc.n_bins
    cases["bin_range"] = good[:28] + a.astype("<u4").tobytes()
    a = w.copy()
    a[w0 + 1] = 0
    cases["zero_count"] = good[:28] + a.astype("<u4").tobytes()
    q = int(np.argmax(np.diff(sc.offsets) > 1))
    if np.diff(sc.offsets)[q] > 1:
        e0q = int(sc.offsets[q])
        wq = q + 1 + 2 * e0q
        a = w.copy()
        a[wq + 2] = a[wq]  # second bin == first bin
        cases["not_increasing"] = good[:28] + a.astype("<u4").tobytes()
    return cases


@pytest.mark.parametrize("name", G.SCENE_NAMES)
def test_encoder_matches_reference(name):
    if not O.ref_available():
        pytest.skip("reference library not built")
    sc, _, _ = G.scene(name)
    assert encode_spcb(sc) == _ref_encode(sc)


def test_reference_rejects_the_bad_cases():
    if not O.ref_available():
        pytest.skip("reference library not built")
    sc, _, _ = G.scene("small_s3")
    for kind, data in _bad_cases(sc).items():
        assert _ref_decode_error(data) is not None, kind


@pytest.mark.gpu
@pytest.mark.parametrize("name", G.SCENE_NAMES)
def test_device_decode_matches_host_path(gpu, name):
    sc, cfg, _ = G.scene(name)
    gpu.set_scene(sc)
    a = gpu.reconstruct(cfg)
    gpu.set_cube_spcb(encode_spcb(sc))
    b = gpu.reconstruct(cfg)
    assert np.array_equal(a["points"], b["points"])
    assert np.array_equal(a["background"], b["background"])
    assert np.array_equal(a["trace"], b["trace"])


@pytest.mark.gpu
def test_device_decode_errors(gpu):
    from paper_1905_06700_b200.rt3d import Rt3dError
    sc, cfg, _ = G.scene("small_s3")
    gpu.set_scene(sc)
    expect = {
        "magic": "SPCB: bad magic", "version": "SPCB: unsupported version 2",
        "zero": "SPCB: zero dimension", "trailing": "SPCB: trailing bytes",
        "truncated_bin": "SPCB: truncated while reading event bin",
        "truncated_value": "SPCB: truncated while reading event value",
        "truncated_header": "SPCB: truncated while reading bin_width",
        "bin_range": "cube: bin out of range at pixel", "zero_count": "cube: zero count at pixel",
        "not_increasing": "cube: bins not strictly increasing at pixel",
    }
    for kind, data in _bad_cases(sc).items():
        with pytest.raises(Rt3dError) as ei:
            gpu.set_cube_spcb(data)
        assert ei.value.status == 2, kind          # RT3D_ERR_FORMAT
        assert expect[kind] in str(ei.value), (kind, str(ei.value))
    gpu.set_cube_spcb(encode_spcb(sc))             # a good cube afterwards
    gpu.reconstruct(cfg)


@pytest.mark.gpu
def test_set_cube_validation_errors(gpu):
    """rt3d_set_cube applies PhotonCube::validate (cube.hpp:84-112) to the
    caller's CSR: each violation is RT3D_ERR_FORMAT with the reference's
    message, and the session stays usable."""
    import copy
    from paper_1905_06700_b200.rt3d import Rt3dError
    sc, cfg, _ = G.scene("small_s3")
    gpu.set_scene(sc)
    p = int(np.argmax(np.diff(sc.offsets.astype(np.int64)) >= 2))   # a pixel with 2+ events
    k = int(sc.offsets[p])

    def bad(mut):
        b = copy.copy(sc)
        b.offsets, b.events = sc.offsets.copy(), sc.events.copy()
        mut(b)
        return b

    cases = {
        "cube: non-positive dimensions": bad(lambda b: setattr(b, "n_bins", 0)),
        "cube: bad offset table": bad(lambda b: b.offsets.__setitem__(-1, b.offsets[-1] - 1)),
        "cube: bins not strictly increasing at pixel": bad(
            lambda b: b.events.__setitem__(k + 1, (b.events[k]["bin"], 1))),
        "cube: bin out of range at pixel": bad(
            lambda b: b.events.__setitem__(k + 1, (b.n_bins, 1))),
        "cube: zero count at pixel": bad(lambda b: b.events.__setitem__(k, (b.events[k]["bin"], 0))),
    }
    # a negative range at the first pixel q whose range starts at event >= 2
    q = int(np.argmax(sc.offsets[:-1] >= 2))
    neg = bad(lambda b: b.offsets.__setitem__(q + 1, b.offsets[q] - 1))
    with pytest.raises(Rt3dError) as ei:
        gpu.set_cube(neg)
    assert ei.value.status == 2
    assert str(ei.value).rstrip().endswith(f"cube: negative event range at pixel {q}"), str(ei.value)
    for msg, b in cases.items():
        with pytest.raises(Rt3dError) as ei:
            gpu.set_cube(b)
        assert ei.value.status == 2, msg           # RT3D_ERR_FORMAT
        assert msg in str(ei.value), (msg, str(ei.value))
        if "pixel" in msg:
            assert str(ei.value).rstrip().endswith(f"pixel {p}"), str(ei.value)
    gpu.set_cube(sc)                               # a good cube afterwards
    rep = gpu.reconstruct(cfg)
    assert len(rep["points"]) > 0
