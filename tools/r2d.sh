timeout 600 python -m pytest tests/test_parity_configs.py -q -x -k "D" > gpurun_out/r2d_parityD.log 2>&1; tail -3 gpurun_out/r2d_parityD.log
CHECK_ITERS=0 timeout 900 python tools/bench_configs.py 3 D E > gpurun_out/r2d_g1.jsonl 2> gpurun_out/r2d_g1.err; tail -2 gpurun_out/r2d_g1.err; cat gpurun_out/r2d_g1.jsonl
RT3D_GSZ=32 CHECK_ITERS=0 timeout 900 python tools/bench_configs.py 3 D > gpurun_out/r2d_g32.jsonl 2>&1; cat gpurun_out/r2d_g32.jsonl | tail -2
timeout 600 python - > gpurun_out/r2d_same.log 2>&1 <<'PY'
import os, sys, subprocess, json
sys.path.insert(0, "tools"); sys.path.insert(0, "tests")
import numpy as np
import workloads as W
from scenegen.scene import simulate
from paper_1905_06700_b200.rt3d import Session
name, spec, seed, cfg = W.config_d()
cfg.max_iters = 4
sc = simulate(spec, seed)
with Session(0) as s:
    s.set_scene(sc)
    a = s.reconstruct(cfg)
np.save("/tmp/d_g1.npy", a["points"]); np.save("/tmp/d_g1_bg.npy", a["background"])
print("g1", len(a["points"]), a["trace"][-1])
PY
RT3D_GSZ=32 timeout 600 python - >> gpurun_out/r2d_same.log 2>&1 <<'PY'
import sys
sys.path.insert(0, "tools")
import numpy as np
import workloads as W
from scenegen.scene import simulate
from paper_1905_06700_b200.rt3d import Session
name, spec, seed, cfg = W.config_d()
cfg.max_iters = 4
sc = simulate(spec, seed)
with Session(0) as s:
    s.set_scene(sc)
    a = s.reconstruct(cfg)
b = np.load("/tmp/d_g1.npy"); bb = np.load("/tmp/d_g1_bg.npy")
print("g32", len(a["points"]), a["trace"][-1], "identical", np.array_equal(a["points"], b), np.array_equal(a["background"], bb))
PY
cat gpurun_out/r2d_same.log
