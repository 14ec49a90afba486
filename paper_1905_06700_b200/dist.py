"""Multi-GPU host logic.

Frames are independent: frame f of a stream goes to rank f mod N and no
collective touches the data path (video, config C; replicas for config B).

Row bands (large arrays, config E): the pixel range is split at the nodes of
parallel::pairwise_sum's recursion (parallel.hpp:52-61) at depth log2(N), so
each rank's band sum is an exact subtree and combining the gathered band sums
with the same tree reproduces the single-GPU nll bit for bit, whatever N.
"""
from __future__ import annotations

import os
from typing import Dict, List, Sequence, Tuple


def frames_for_rank(n_frames: int, rank: int, world: int) -> List[int]:
    """Frame f -> rank f mod world."""
    return list(range(rank, n_frames, world))


def band_bounds(n: int, world: int) -> List[Tuple[int, int]]:
    """[lo, hi) of the depth-log2(world) nodes of pairwise_sum's tree over n
    elements (world a power of two; a node of <= 8 elements is not split, so
    ranks past it get empty bands)."""
    if world < 1 or world & (world - 1):
        raise ValueError("world size must be a power of two")
    nodes = [(0, n)]
    while len(nodes) < world:
        nxt = []
        for lo, hi in nodes:
            size = hi - lo
            if size <= 8:
                nxt += [(lo, hi), (hi, hi)]
            else:
                h = size // 2
                nxt += [(lo, lo + h), (lo + h, hi)]
        nodes = nxt
    return nodes


def combine_band_sums(sums: Sequence[float], sizes: Sequence[int]) -> float:
    """The top of pairwise_sum's tree over the band sums (depth-ordered
    pairwise combination; leaves that were not split keep their own sum)."""
    vals = list(sums)
    szs = list(sizes)
    while len(vals) > 1:
        nv, ns = [], []
        for k in range(0, len(vals), 2):
            a, b = vals[k], vals[k + 1]
            if szs[k] + szs[k + 1] <= 8 and szs[k + 1] == 0:
                nv.append(a)  # an unsplit leaf (the partner is the empty half)
            else:
                nv.append(a + b)
            ns.append(szs[k] + szs[k + 1])
        vals, szs = nv, ns
    return vals[0] if vals else 0.0


def halo_ranges(bounds: Sequence[Tuple[int, int]], rank: int, halo_px: int, npix: int):
    """The pixel ranges rank reads from its neighbours before APSS and kNN
    (halo_kernel, rt3d.cu): [(neighbour, lo, hi)], halo_px = halo rows x cols."""
    lo, hi = bounds[rank]
    out = []
    if rank > 0:
        out.append((rank - 1, max(lo - halo_px, 0), lo))
    if rank + 1 < len(bounds):
        out.append((rank + 1, hi, min(hi + halo_px, npix)))
    return out


def exchange_halos(bo, values: dict, bounds, rank: int, halo_px: int):
    """Host mirror of halo_kernel over torch.distributed point-to-point
    (gloo on CPU): every band keeps full-size arrays in the global index
    space; it receives its neighbours' halo pixels' bucket offsets `bo`
    (npix + 1) and, for their points, each array in `values`, at the same
    indices.  Both sides derive the point ranges from the sender's offsets,
    so a band first receives the offsets, then the point slices."""
    import torch
    import torch.distributed as dist
    npix = len(bo) - 1
    me = halo_ranges(bounds, rank, halo_px, npix)
    ops = []
    # what my neighbours read from me (their halo ranges inside my band)
    sends = []
    for nb in (rank - 1, rank + 1):
        if 0 <= nb < len(bounds):
            for owner, a, b in halo_ranges(bounds, nb, halo_px, npix):
                if owner == rank:
                    sends.append((nb, a, b))
    for nb, a, b in sends:
        ops.append(dist.isend(torch.from_numpy(bo[a:b + 1].copy()), nb))
    recvd = []
    for owner, a, b in me:
        buf = torch.empty(b - a + 1, dtype=torch.from_numpy(bo[:1]).dtype)
        ops.append(dist.irecv(buf, owner))
        recvd.append((owner, a, b, buf))
    for op in ops:
        op.wait()
    ops = []
    for owner, a, b, buf in recvd:
        if owner < rank:
            bo[a:b] = buf.numpy()[:-1]      # bo[lo] is ours
        else:
            bo[a + 1:b + 1] = buf.numpy()[1:]
    for nb, a, b in sends:
        n0, n1 = int(bo[a]), int(bo[b])
        for k in sorted(values):
            ops.append(dist.isend(torch.from_numpy(values[k][n0:n1].copy()), nb))
    pending = []
    for owner, a, b, _ in recvd:
        n0, n1 = int(bo[a]), int(bo[b])
        for k in sorted(values):
            buf = torch.empty(n1 - n0, dtype=torch.from_numpy(values[k][:1]).dtype)
            ops.append(dist.irecv(buf, owner))
            pending.append((k, n0, n1, buf))
    for op in ops:
        op.wait()
    for k, n0, n1, buf in pending:
        values[k][n0:n1] = buf.numpy()


def env_rank() -> Tuple[int, int, int]:
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def gather_objects(obj, world: int):
    """all_gather_object over the default process group (world 1: [obj])."""
    if world == 1:
        return [obj]
    import torch.distributed as dist
    out: List = [None] * world
    dist.all_gather_object(out, obj)
    return out


def merge_frame_results(per_rank: Sequence[Dict[int, object]]) -> Dict[int, object]:
    merged: Dict[int, object] = {}
    for d in per_rank:
        for f, v in d.items():
            if f in merged:
                raise ValueError(f"frame {f} reconstructed twice")
            merged[f] = v
    return dict(sorted(merged.items()))
