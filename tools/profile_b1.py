"""One single-frame config-B reconstruct between cudaProfilerStart/Stop
(after a warm-up frame), for `ncu --profile-from-start off -k regex:... `."""
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
name, spec, seed, cfg = W.CONFIGS[key]()
with Session(0) as s:
    s.set_scene(simulate(spec, seed))
    s.reconstruct_async(cfg)
    s.synchronize()
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    s.reconstruct_async(cfg)
    s.synchronize()
    torch.cuda.profiler.stop()
print("profiled one frame")
