"""FFT background low-pass timings: the standalone operator
(rt3d_fft_lowpass_filter, wall clock incl. copies) at 141^2 (direct DFT),
256^2 and 1024^2 (radix 2), and config D reconstructions with the FFT
background against the identity background (CUDA events)."""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_1905_06700_b200.rt3d import Session  # noqa: E402
from scenegen.scene import simulate  # noqa: E402

with Session(0) as s:
    for n in (141, 256, 1024):
        img = np.random.default_rng(n).uniform(0, 1, (n, n))
        s.fft_lowpass(img, 0.5)
        t0 = time.perf_counter()
        for _ in range(5):
            s.fft_lowpass(img, 0.5)
        print(json.dumps({"op": "fft_lowpass_filter", "n": n,
                          "ms": 1e3 * (time.perf_counter() - t0) / 5}), flush=True)
    name, spec, seed, cfg = W.config_d()
    cfg.max_iters = 10
    sc = simulate(spec, seed)
    s.set_scene(sc)
    stream = torch.cuda.ExternalStream(s.stream_ptr, device=torch.device("cuda", 0))
    for mode in (0, 1):
        cfg.background_mode = mode
        s.reconstruct_async(cfg)
        s.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            a.record(stream)
            s.reconstruct_async(cfg)
            b.record(stream)
        stream.synchronize()
        print(json.dumps({"op": "reconstruct D 10 iterations", "background_mode": mode,
                          "ms": a.elapsed_time(b)}), flush=True)
