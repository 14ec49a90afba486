"""One batch of 8 config-B frames (bench.py's step) between
cudaProfilerStart/Stop, for `ncu --profile-from-start off ...`; a warm-up
batch first (module load, buffers, the CUDA graph)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_1905_06700_b200.rt3d import Session  # noqa: E402
from scenegen.scene import simulate  # noqa: E402

name, spec, seed, cfg = W.config_b()
ss = [Session(0) for _ in range(8)]
for k, s in enumerate(ss):
    s.set_scene(simulate(spec, seed + k))
Session.reconstruct_batch_async(ss, cfg)
ss[0].synchronize()
torch.cuda.synchronize()
torch.cuda.profiler.start()
Session.reconstruct_batch_async(ss, cfg)
ss[0].synchronize()
torch.cuda.profiler.stop()
for s in ss:
    s.close()
print("profiled one batch of 8 frames")
