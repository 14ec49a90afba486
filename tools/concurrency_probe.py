"""Throughput of S sessions (streams) each with F frames in flight, config B.
usage: RT3D_BLOCKS_PER_SM=1 python tools/concurrency_probe.py S N"""
import sys, time, os
sys.path.insert(0, '.')
import numpy as np
import bench
from paper_1905_06700_b200.rt3d import Session
from scenegen.scene import simulate
S = int(sys.argv[1]); N = int(sys.argv[2])
spec, seed, cfg, _ = bench.config_b()
sc = simulate(spec, seed)
ss = [Session(0) for _ in range(S)]
for s in ss:
    s.set_scene(sc)
# warm: two frames per session (both slots / graphs)
for s in ss:
    for _ in range(2):
        s.frame_collect(s.frame_submit(sc, cfg))
t0 = time.perf_counter()
pend = []
for k in range(N):
    s = ss[k % S]
    if len(pend) >= 2 * S:
        ps, pt = pend.pop(0)
        ps.frame_collect(pt)
    pend.append((s, s.frame_submit(sc, cfg)))
for ps, pt in pend:
    p, b, r = ps.frame_collect(pt)
dt = time.perf_counter() - t0
print(f"sessions={S} blocks/SM={os.environ.get('RT3D_BLOCKS_PER_SM','2')} frames={N} fps={N/dt:.1f}", flush=True)
