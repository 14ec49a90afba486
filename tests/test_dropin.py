"""The C++ drop-in (include/splidar/b200.hpp) against the reference's own
functions, through tests/cpp/dropin_check.cpp (built by oracle/Makefile where
the reference headers exist; the binary travels to the GPU box)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "dropin_check")
REF_INC = "/root/reference/proj/include"


@pytest.mark.skipif(not os.path.isdir(REF_INC), reason="reference headers absent")
def test_dropin_header_compiles_warning_free():
    src = os.path.join(ROOT, "tests", "cpp", "dropin_check.cpp")
    r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-Wall", "-Wextra",
                        "-I" + REF_INC, "-I/root/reference/proj/tests",
                        "-I" + os.path.join(ROOT, "oracle", "shim"),
                        "-I" + os.path.join(ROOT, "include"),
                        "-isystem", os.path.join(ROOT, "oracle", "shim"), src],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]
    own = [l for l in r.stderr.splitlines() if "b200.hpp" in l and "warning" in l]
    assert not own, "\n".join(own)


def test_dropin_binary_fails_loudly_without_device():
    if not os.path.exists(BIN):
        pytest.skip("dropin_check not built")
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=60)
    assert r.returncode != 0
    assert "no CUDA device" in r.stderr


@pytest.mark.gpu
def test_dropin_matches_reference():
    if not os.path.exists(BIN):
        pytest.skip("dropin_check not built (reference headers were absent at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0 and "DROPIN OK" in r.stdout, r.stdout[-4000:] + r.stderr[-2000:]
