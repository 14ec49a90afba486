"""CPU, world size 2 over gloo: the host side of the multi-GPU paths.
 - frames sharded across ranks (frame f -> rank f mod N) gather to exactly
   the single-process result;
 - row bands at pairwise_sum's split points reproduce the single-rank nll
   reduction bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1905_06700_b200 import dist as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _frame_digest(f):
    """Stand-in per-frame result: the C oracle's reconstruct of a small
    synthetic frame (test infrastructure as the checker)."""
    import oracle_lib as O
    from paper_1905_06700_b200.abi import Config
    from scenegen.scene import SceneSpec, SurfaceSpec, simulate
    spec = SceneSpec(rows=6, cols=6, bins=120, bin_resolution_m=0.01, pixel_pitch_m=0.02,
                     target_ppp=20, target_sbr=5,
                     surfaces=[SurfaceSpec(depth_m=0.5 + 0.01 * f)])
    sc = simulate(spec, 1000 + f, threads=1)
    r = O.reconstruct(sc, Config(max_iters=2, apss_radius=0.05, knn_k=5, r_min=0.1,
                                 init_max_returns=2, init_min_separation=6, stop_tol=0.0))
    return r["points"].tobytes() + r["background"].tobytes()


def _worker(rank, world, port, n_frames, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = {f: _frame_digest(f) for f in D.frames_for_rank(n_frames, rank, world)}
    merged = D.merge_frame_results(D.gather_objects(mine, world))
    # row bands of a partial-nll vector
    rng = np.random.default_rng(7)
    part = rng.standard_normal(19881) * 1e3
    bounds = D.band_bounds(len(part), world)
    import oracle_lib as O
    lo, hi = bounds[rank]
    band = np.ascontiguousarray(part[lo:hi])
    s = O.oracle().oracle_pairwise_sum(band.ctypes.data_as(O.P(O._dbl)), len(band)) if len(band) else 0.0
    sums = D.gather_objects(s, world)
    total = D.combine_band_sums(sums, [h - l for l, h in bounds])
    if rank == 0:
        q.put((sorted(merged), [merged[f] for f in sorted(merged)], total))
    dist.barrier()
    dist.destroy_process_group()


def test_frames_and_bands_world2():
    n_frames, world = 5, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_frames, q)) for r in range(world)]
    for p in procs:
        p.start()
    frames, digests, total = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert frames == list(range(n_frames))
    for f in range(n_frames):
        assert digests[f] == _frame_digest(f)
    import oracle_lib as O
    rng = np.random.default_rng(7)
    part = np.ascontiguousarray(rng.standard_normal(19881) * 1e3)
    single = O.oracle().oracle_pairwise_sum(part.ctypes.data_as(O.P(O._dbl)), len(part))
    assert total == single  # bitwise


@pytest.mark.parametrize("n", [1, 5, 8, 9, 17, 144, 19881, 1 << 20])
@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_band_split_reproduces_pairwise_sum(n, world):
    import oracle_lib as O
    rng = np.random.default_rng(n + world)
    v = np.ascontiguousarray(rng.standard_normal(n) * 1e5)
    b = D.band_bounds(n, world)
    assert b[0][0] == 0 and b[-1][1] == n
    sums = []
    for lo, hi in b:
        seg = np.ascontiguousarray(v[lo:hi])
        sums.append(O.oracle().oracle_pairwise_sum(seg.ctypes.data_as(O.P(O._dbl)), len(seg))
                    if len(seg) else 0.0)
    got = D.combine_band_sums(sums, [hi - lo for lo, hi in b])
    assert got == O.oracle().oracle_pairwise_sum(v.ctypes.data_as(O.P(O._dbl)), n)


def test_frames_for_rank_partition():
    for world in (1, 2, 4, 8):
        got = sorted(f for r in range(world) for f in D.frames_for_rank(37, r, world))
        assert got == list(range(37))


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_band_plan_matches_host_bounds(world):
    """rt3d_band_plan (librt3d, host only) splits at pairwise_sum's nodes
    exactly as dist.band_bounds does; every halo lies in the neighbour band."""
    from paper_1905_06700_b200 import rt3d
    rows = cols = 1024
    plan, hrows = rt3d.band_plan(rows, cols, 1, 0.02, 0.16, world)
    assert plan == D.band_bounds(rows * cols, world)
    assert hrows == 9          # floor(0.16 / 0.02) + 1 fine pixels, superres 1
    for r in range(world):
        for owner, a, b in D.halo_ranges(plan, r, hrows * cols, rows * cols):
            lo, hi = plan[owner]
            assert lo <= a <= b <= hi


def test_band_plan_rejects_partial_rows():
    from paper_1905_06700_b200 import rt3d
    with pytest.raises(rt3d.Rt3dError):
        rt3d.band_plan(141, 141, 1, 0.0025, 0.02, 2)   # config B: the halves split a row


def _halo_worker(rank, world, port, q):
    """Each rank holds its band of a random pixel-major cloud in full-size
    arrays (global indices), exchanges halos with its neighbours over gloo
    following the band plan, and checks own band + halo rows against the
    global arrays."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1905_06700_b200 import rt3d
    rows, cols = 64, 48
    plan, hrows = rt3d.band_plan(rows, cols, 1, 0.02, 0.1, world)
    npix = rows * cols
    rng = np.random.default_rng(11)
    counts = rng.integers(0, 4, npix)
    bo_all = np.zeros(npix + 1, np.uint32)
    np.cumsum(counts, out=bo_all[1:])
    t_all = rng.standard_normal(int(bo_all[-1]))
    r_all = rng.random(int(bo_all[-1]))
    lo, hi = plan[rank]
    bo = np.zeros_like(bo_all)
    bo[lo:hi + 1] = bo_all[lo:hi + 1]                 # what the band's own scan wrote
    t = np.full_like(t_all, np.nan)
    r = np.full_like(r_all, np.nan)
    a, b = bo_all[lo], bo_all[hi]
    t[a:b], r[a:b] = t_all[a:b], r_all[a:b]
    D.exchange_halos(bo, {"t": t, "r": r}, plan, rank, hrows * cols)
    ok = True
    for owner, x0, x1 in D.halo_ranges(plan, rank, hrows * cols, npix):
        ok &= np.array_equal(bo[x0:x1 + 1], bo_all[x0:x1 + 1])
        n0, n1 = bo_all[x0], bo_all[x1]
        ok &= np.array_equal(t[n0:n1], t_all[n0:n1]) and np.array_equal(r[n0:n1], r_all[n0:n1])
    q.put((rank, bool(ok)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_halo_exchange_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_halo_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = sorted(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got == [(r, True) for r in range(world)]
