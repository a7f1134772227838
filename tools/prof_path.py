"""ncu driver: load a converged raw C3 field and run the path kernels 3 times."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1903_07441_b200 import Planner, band_cfg, warp_cfg
from scenes import scene_c3
sc = scene_c3(0)
pl = Planner(sc.W, sc.H, 1, sc.cell_size, sc.origin, 0, torch.cuda.current_stream().cuda_stream)
pl.set_static(sc.static)
pl.set_obstacles(0, sc.robot, sc.goal, sc.tracks, warp_cfg(), warm=0)
pl.set_field(np.load(sys.argv[1]))
for _ in range(3):
    s, cells, *_ = pl.extract_path(0, band_cfg(50, 40000, 80000))
print("walk", s, len(cells))
