"""One batch of 8 frames of a workload (default config B) between
cudaProfilerStart/Stop, for `ncu --profile-from-start off ...`; a warm-up
batch first (module load, buffers, the CUDA graph).
usage: python tools/profile_batch.py [B|C] [frames]"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_1905_06700_b200.rt3d import Session  # noqa: E402
from scenegen.scene import simulate  # noqa: E402

key = sys.argv[1] if len(sys.argv) > 1 else "B"
nf = int(sys.argv[2]) if len(sys.argv) > 2 else 8
name, spec, seed, cfg = W.CONFIGS[key]()
ss = [Session(0) for _ in range(nf)]
for k, s in enumerate(ss):
    if key == "C":
        _, spec, seed, _ = W.config_c(k)
        s.set_scene(simulate(spec, seed))
    else:
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
print(f"profiled one batch of {nf} frames")
