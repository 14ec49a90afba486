"""GPU: the denoisers on arbitrary clouds (rt3d_apss_project,
rt3d_knn_intensity_filter, rt3d_prune; denoise.hpp:159-248) through the
device SpatialIndex (a cell grid sorted by the reference's cell key, 27-cell
queries merged in ascending point index, spatial_index.hpp:18-77) against the
C oracle and the reference itself, on clouds spanning many cells, with a
separate index cloud, a cell larger than the radius, and collinear and
isolated points."""
import numpy as np
import pytest

import oracle_lib as O
from paper_1905_06700_b200.abi import POINT_DTYPE

pytestmark = pytest.mark.gpu


def _cloud(n, seed):
    rng = np.random.default_rng(seed)
    c = np.zeros(n, POINT_DTYPE)
    # a noisy sphere of radius 1, a tilted plane, a line and a few strays
    k = n // 3
    u = rng.normal(size=(k, 3))
    u /= np.linalg.norm(u, axis=1)[:, None]
    sph = u * (1.0 + 0.01 * rng.normal(size=(k, 1))) + np.array([3.0, 0.0, 0.0])
    xy = rng.uniform(-2.0, 2.0, size=(k, 2))
    pla = np.column_stack([xy[:, 0], xy[:, 1], 0.3 * xy[:, 0] + 0.005 * rng.normal(size=k)])
    m = n - 2 * k - 10
    lin = np.column_stack([np.linspace(-4, -2, m), np.zeros(m), np.zeros(m)])
    stray = rng.uniform(-8, 8, size=(10, 3))
    xyz = np.vstack([sph, pla, lin, stray])
    perm = rng.permutation(n)      # interleave, so balls mix far-apart indices
    xyz = xyz[perm]
    c["x"], c["y"], c["z"] = xyz[:, 0], xyz[:, 1], xyz[:, 2]
    c["intensity"] = rng.uniform(0.0, 5.0, n)
    c["i"] = np.arange(n) % 97
    c["j"] = np.arange(n) % 89
    return c


@pytest.mark.parametrize("n,radius,cell", [(3000, 0.35, 0.35), (12000, 0.2, 0.3)])
def test_apss_general_cloud_matches_oracle(gpu, n, radius, cell):
    cloud = _cloud(n, n)
    got = gpu.apss_project(cloud, radius, cell=cell)
    exp = O.apss_project(cloud, radius, cell=cell, impl="oracle")
    assert np.array_equal(got["flags"], exp["flags"])
    assert np.any(got["flags"] & 1) and np.any(got["flags"] & 4)   # isolated, degenerate
    for k in "xyz":
        assert np.max(np.abs(got[k] - exp[k])) <= 1e-12, k
    if O.ref_available():   # the reference: flags equal, positions within its eigen-solver's 1e-9
        ref = O.apss_project(cloud, radius, cell=cell, impl="ref")
        assert np.array_equal(got["flags"], ref["flags"])
        for k in "xyz":
            assert np.max(np.abs(got[k] - ref[k])) <= 1e-9, k


@pytest.mark.parametrize("n,k,radius,cell", [(3000, 9, 0.35, 0.35), (12000, 5, 0.2, 0.3),
                                            (12000, 40, 0.3, 0.3)])
def test_knn_general_cloud_matches_oracle_and_reference(gpu, n, k, radius, cell):
    cloud = _cloud(n, n + k)
    got = gpu.knn_filter(cloud, k, radius, cell=cell)
    assert np.array_equal(got, O.knn_filter(cloud, k, radius, cell=cell, impl="oracle"))
    if O.ref_available():
        assert np.array_equal(got, O.knn_filter(cloud, k, radius, cell=cell, impl="ref"))


def test_denoisers_with_a_separate_index_cloud(gpu):
    cloud, index = _cloud(2000, 5), _cloud(5000, 6)
    got = gpu.knn_filter(cloud, 7, 0.3, index=index)
    from paper_1905_06700_b200.abi import Point, ptr
    import ctypes as C
    exp = np.zeros(len(cloud), POINT_DTYPE)
    rc = O.oracle().oracle_knn_intensity_filter(ptr(cloud, Point), len(cloud), 7, ptr(index, Point),
                                                len(index), 0.3, 0.3, ptr(exp, Point))
    assert rc == 0
    assert np.array_equal(got, exp)


@pytest.mark.parametrize("n", [1, 255, 256, 257, 100000])
def test_prune_general_cloud(gpu, n):
    cloud = _cloud(max(n, 60), n)[:n]
    for r_min in (0.0, 2.5, 6.0):
        got = gpu.prune(cloud, r_min)
        assert np.array_equal(got, cloud[cloud["intensity"] >= r_min])
