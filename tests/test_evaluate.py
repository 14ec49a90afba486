"""evaluate (eval.hpp:33-87): the oracle against the reference's golden
outputs (tests/golden/evaluate.npz, made by make_golden.py from
oracle/_ref), and the GPU rt3d_evaluate against both, bit for bit."""
import numpy as np
import pytest

import oracle_lib as L

GOLD = L.ROOT / "tests" / "golden" / "evaluate.npz"
FIELDS = ("recall", "false_point_rate", "depth_rmse", "intensity_mae", "n_truth", "n_est",
          "n_matched")


def cases():
    g = np.load(GOLD)
    return [(str(n), g[f"{n}_est"], g[f"{n}_truth"], *map(float, g[f"{n}_tp"]), g[f"{n}_out"])
            for n in g["names"]]


def bits(a):
    return np.asarray(a, np.float64).view(np.uint64)


@pytest.mark.parametrize("case", cases(), ids=lambda c: c[0])
def test_oracle_evaluate_matches_golden(case):
    _, e, t, tau, pitch, want = case
    got, rc = L.evaluate(e, t, tau, pitch, "oracle")
    assert rc == 0
    assert (bits(got) == bits(want)).all(), (got, want)


def test_oracle_evaluate_rejects_bad_args():
    e = np.zeros(1, L.POINT_DTYPE)
    assert L.evaluate(e, e, 0.0, 1.0, "oracle")[1] == 1
    assert L.evaluate(e, e, 1.0, -1.0, "oracle")[1] == 1


@pytest.mark.skipif(not L.ref_available(), reason="oracle/_ref not built")
def test_oracle_evaluate_matches_reference_random():
    rng = np.random.default_rng(7)
    for trial in range(20):
        n, m = rng.integers(0, 400, 2)
        e = np.zeros(n, L.POINT_DTYPE)
        t = np.zeros(m, L.POINT_DTYPE)
        for c in (e, t):
            c["x"], c["y"] = rng.uniform(-0.3, 0.3, (2, len(c)))
            c["z"] = np.round(rng.uniform(0, 1, len(c)), 2)
            c["intensity"] = rng.uniform(0, 2, len(c))
        tau, pitch = rng.uniform(0.01, 0.2), rng.uniform(0.02, 0.2)
        a, ra = L.evaluate(e, t, tau, pitch, "oracle")
        b, rb = L.evaluate(e, t, tau, pitch, "ref")
        assert ra == rb == 0
        assert (bits(a) == bits(b)).all(), (trial, a, b)


@pytest.mark.gpu
@pytest.mark.parametrize("case", cases(), ids=lambda c: c[0])
def test_gpu_evaluate_bit_exact(gpu, case):
    _, e, t, tau, pitch, want = case
    got = gpu.evaluate(e, t, tau, pitch)
    assert (bits([got[k] for k in FIELDS]) == bits(want)).all(), (got, want)


@pytest.mark.gpu
def test_gpu_evaluate_random_vs_oracle(gpu):
    rng = np.random.default_rng(11)
    for trial in range(10):
        n, m = rng.integers(1, 5000, 2)
        e = np.zeros(n, L.POINT_DTYPE)
        t = np.zeros(m, L.POINT_DTYPE)
        for c in (e, t):
            c["x"], c["y"] = rng.uniform(-2, 2, (2, len(c)))
            c["z"] = np.round(rng.uniform(0, 1, len(c)), 3)
            c["intensity"] = rng.uniform(0, 2, len(c))
        want, rc = L.evaluate(e, t, 0.05, 0.1, "oracle")
        got = gpu.evaluate(e, t, 0.05, 0.1)
        assert (bits([got[k] for k in FIELDS]) == bits(want)).all(), (trial, got, want)


@pytest.mark.gpu
def test_gpu_evaluate_errors(gpu):
    from paper_1905_06700_b200.rt3d import Rt3dError
    e = np.zeros(3, L.POINT_DTYPE)
    with pytest.raises(Rt3dError, match="evaluate: tau must be positive"):
        gpu.evaluate(e, e, 0.0, 1.0)
    with pytest.raises(Rt3dError, match="evaluate: pitch must be positive"):
        gpu.evaluate(e, e, 0.1, 0.0)
    big = np.zeros(100, L.POINT_DTYPE)  # one column holding 100 estimates
    with pytest.raises(Rt3dError, match="more than 64"):
        gpu.evaluate(big, e, 0.1, 1.0)
