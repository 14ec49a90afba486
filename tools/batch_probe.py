"""Frames/s of batched reconstructs (rt3d_reconstruct_batch) for configs B
and C at batch sizes 1, 2, 4, 8 (BATCHES=...): CUDA events around each
batch, inputs resident, L2 flushed between batches.  KT=1 adds the per-class
kernel times per frame."""
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_1905_06700_b200.rt3d import Session  # noqa: E402
from scenegen.scene import simulate  # noqa: E402

keys = sys.argv[1:] or ["B", "C"]
flush = torch.empty(64 * 2 ** 20, dtype=torch.float32, device="cuda:0")
for key in keys:
    name, spec, seed, cfg = W.CONFIGS[key]()
    cubes = [simulate(W.config_c(f)[1], 1000 + f) for f in range(32)] if key == "C" else \
        [simulate(spec, seed)] * 32
    for n in [int(x) for x in os.environ.get("BATCHES", "1,2,4,8").split(",")]:
        ss = [Session(0) for _ in range(n)]
        for s, c in zip(ss, cubes):
            s.set_scene(c)
        stream = torch.cuda.ExternalStream(ss[0].stream_ptr, device=torch.device("cuda", 0))
        try:
            for _ in range(3):
                Session.reconstruct_batch_async(ss, cfg)
            ss[0].synchronize()
            K = 10
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                  for _ in range(K)]
            with torch.cuda.stream(stream):
                for k in range(K):
                    flush.zero_()
                    ev[k][0].record(stream)
                    Session.reconstruct_batch_async(ss, cfg)
                    ev[k][1].record(stream)
            stream.synchronize()
            ms = sum(a.elapsed_time(b) for a, b in ev) / K
            print(json.dumps({"config": key, "batch": n, "ms_per_batch": ms,
                              "frames_per_s": 1e3 * n / ms}), flush=True)
            if os.environ.get("KT"):  # per-class kernel ms per frame (events around each launch)
                ss[0].time_kernels(True)
                for _ in range(K):
                    Session.reconstruct_batch_async(ss, cfg)
                kt = ss[0].kernel_times()
                ss[0].time_kernels(False)
                print(json.dumps({"config": key, "batch": n, "kernel_ms_per_frame": {
                    k: round(v[0] / (K * n), 4) for k, v in kt.items() if v[1]}}), flush=True)
        except Exception as e:  # noqa: BLE001
            print(json.dumps({"config": key, "batch": n, "error": str(e)}), flush=True)
        finally:
            for s in ss:
                s.close()
