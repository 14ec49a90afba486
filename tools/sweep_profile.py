"""Per-transition timing of the in-kernel profile stamps of one frame of a
workload (default config B; sweep sub-phases 100..113 included when compiled
in: block 0's view, so 101->102 is the grid barrier's wait).
usage: python tools/sweep_profile.py [A|B|C|D]  (sub-phases need a build with
  make -C paper_1905_06700_b200/csrc EXTRA=-DRT3D_SWEEP_PROF)"""
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))
import workloads as W  # noqa: E402
from paper_1905_06700_b200.rt3d import Session  # noqa: E402
from scenegen.scene import simulate  # noqa: E402

_, spec, seed, cfg = W.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "B"]()
sc = simulate(spec, seed)
with Session(0) as s:
    s.set_scene(sc)
    s.reconstruct_async(cfg)
    s.synchronize()
    s.profile(True)
    s.reconstruct_async(cfg)
    s.synchronize()
    import ctypes as C
    import numpy as np
    from paper_1905_06700_b200 import rt3d as M
    cap = 1 << 16
    buf = np.zeros(2 * cap, np.uint64)
    n = C.c_uint32()
    M._check(M.lib().rt3d_profile_copy(s.h, M.ptr(buf, M._u64), cap, C.byref(n)))
    pairs = buf[: 2 * n.value].reshape(-1, 2)
    agg = defaultdict(lambda: [0, 0.0])
    names = {k: v for k, v in Session.PHASES.items()}
    prev = None
    for pid, ts in pairs:
        pid, ts = int(pid), int(ts)
        if prev is not None:
            key = f"{names.get(prev[0], prev[0])}->{names.get(pid, pid)}"
            a = agg[key]
            a[0] += 1
            a[1] += (ts - prev[1]) / 1e3
        prev = (pid, ts)
    tot = sum(v[1] for v in agg.values())
    print(f"stamps {n.value}, total {tot:.1f} us")
    for k, (c, us) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:40]:
        print(f"{k:28s} n={c:5d} total={us:9.1f} us  mean={us / c:7.2f} us")
