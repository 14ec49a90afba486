"""GPU parity at the benchmark workloads (BASELINE.json
configs A-D): the CUDA path through the C ABI against the C oracle (full
25-iteration reconstructions, same trajectory) and against the reference
itself (oracle/_ref/libref.so: bit-exact init, then every PALM step from the
reference's own state).  Tolerances are the north star's (tests/parity.py):
depth within 1e-3 bins, intensity within 1e-4 relative, point count within
0.1 %, matched-filter peaks bit-exact.

Inputs: the reference's own simulate_cube (libref) on the workload's
SceneSpec, checked equal to the benchmark's generator.  Config E (1M pixels)
is covered by tests/test_bands.py's band-decomposition identity instead:
the checkers need minutes per iteration there.
"""
import numpy as np
import pytest

import oracle_lib as O
import parity as PY
import workloads as W
from scenegen.scene import simulate

pytestmark = pytest.mark.gpu

needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref/libref.so not built")


def _workload(key, iters=None):
    name, spec, seed, cfg = W.CONFIGS[key]()
    if iters is not None:
        cfg.max_iters = iters
    if O.ref_available():
        sc = O.ref_simulate(W.spec_text(spec), seed)
        ours = simulate(spec, seed)
        assert np.array_equal(sc.offsets, ours.offsets) and np.array_equal(sc.events, ours.events)
    else:
        sc = simulate(spec, seed)
    return sc, cfg


@pytest.mark.parametrize("key,iters", [("A", 25), ("B", 25), ("C", 25), ("D", 3)])
def test_free_running_matches_oracle(gpu, key, iters):
    sc, cfg = _workload(key, iters)
    d = PY.free_running(gpu, sc, cfg, "oracle")
    assert d["iterations"][0] == d["iterations"][1] == iters
    assert PY.within_tolerance(d), d
    assert d["flags_equal"], d
    assert d["backtracks_equal"], d
    assert d["trace_max_rel"] <= 1e-9, d


@needs_ref
@pytest.mark.parametrize("key", ["A", "B", "C", "D"])
def test_init_bit_exact_vs_reference(gpu, key):
    sc, cfg = _workload(key)
    assert PY.init_bitexact(gpu, sc, cfg, "ref")


@needs_ref
@pytest.mark.parametrize("key,iters", [("A", 25), ("B", 25), ("C", 25), ("D", 3)])
def test_every_palm_step_matches_reference(gpu, key, iters):
    sc, cfg = _workload(key, iters)
    w = PY.stepwise(gpu, sc, cfg, "ref")
    assert w["steps"] == iters, w
    assert w["same_cells"] and w["count_rel"] == 0.0, w
    assert w["max_dt_bins"] <= PY.T_TOL_BINS, w
    assert w["max_rel_dr"] <= PY.R_TOL_REL, w
    assert w["flags_equal"] and w["backtracks_equal"], w
    assert w["nll_max_rel"] <= 1e-9, w
