"""CPU: librt3d.so (and the input generator scenegen/libscene.so) load, export
every symbol their headers declare, and refuse to compute without a CUDA device (no CPU fallback)."""
import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

from paper_1905_06700_b200 import abi, rt3d
from scenegen import scene

ROOT = Path(__file__).resolve().parents[1]


def declared(header, where="include"):
    text = (ROOT / where / header).read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(rt3d_[a-z0-9_]+)\s*\(", text)))


def test_librt3d_exports_every_declared_symbol():
    L = rt3d.lib()
    names = declared("rt3d.h")
    assert len(names) >= 30
    for n in names:
        assert hasattr(L, n), n
    assert set(rt3d.EXPORTED) <= set(names)
    assert L.rt3d_abi_version() == 1


def test_libscene_exports_every_declared_symbol():
    L = scene.lib()
    for n in declared("rt3d_scene.h", "scenegen"):
        assert hasattr(L, n), n


def test_struct_layouts_match_the_c_header(tmp_path):
    """ctypes mirrors == the C compiler's layout of include/rt3d.h."""
    import shutil
    import subprocess
    if not shutil.which("gcc"):
        pytest.skip("gcc not available")
    pairs = {"rt3d_point": abi.Point, "rt3d_event": abi.Event, "rt3d_irf": abi.Irf,
             "rt3d_sensor": abi.Sensor, "rt3d_cube": abi.Cube, "rt3d_state_view": abi.StateView,
             "rt3d_init_params": abi.InitParams, "rt3d_apss_params": abi.ApssParams,
             "rt3d_recon_config": abi.ReconConfig, "rt3d_peak": abi.Peak,
             "rt3d_block_diag": abi.BlockDiag, "rt3d_step_diag": abi.StepDiag,
             "rt3d_report": abi.Report}
    src = tmp_path / "sz.c"
    src.write_text('#include "rt3d.h"\n#include <stdio.h>\n#include <stddef.h>\nint main(void){\n' +
                   "".join(f'printf("{k} %zu\\n", sizeof({k}));\n' for k in pairs) +
                   'printf("cfg.r_min %zu\\n", offsetof(rt3d_recon_config, r_min));\n' +
                   'printf("cfg.init %zu\\n", offsetof(rt3d_recon_config, init));\n' +
                   "return 0;}\n")
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-I", str(ROOT / "include"), str(src), "-o", str(exe)], check=True)
    out = dict(l.split() for l in subprocess.run([str(exe)], capture_output=True, text=True,
                                                 check=True).stdout.split("\n") if l)
    for k, t in pairs.items():
        assert int(out[k]) == C.sizeof(t), k
    assert int(out["cfg.r_min"]) == abi.ReconConfig.r_min.offset
    assert int(out["cfg.init"]) == abi.ReconConfig.init.offset
    assert C.sizeof(abi.Point) == 64 == abi.POINT_DTYPE.itemsize
    assert C.sizeof(abi.StepDiag) == abi.STEP_DIAG_DTYPE.itemsize


def test_no_cpu_fallback():
    L = rt3d.lib()
    if L.rt3d_device_count() > 0:
        pytest.skip("a CUDA device is present")
    with pytest.raises(rt3d.Rt3dError) as e:
        rt3d.Session(0)
    assert e.value.status == 7  # RT3D_ERR_NO_DEVICE
