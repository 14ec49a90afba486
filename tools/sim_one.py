import sys, os
sys.path.insert(0, os.getcwd())
import bench
from paper_1905_06700_b200.rt3d import Session
from scenegen.scene import simulate
spec, seed = bench.config_b()[:2]
sc = simulate(spec, seed)
s = Session(0)
s.set_scene(sc)
for _ in range(2):
    s.simulate_cube(sc.truth, sc.background_truth, seed)
print("ok")
