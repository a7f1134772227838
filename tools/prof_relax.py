"""ncu driver for k_rb_tblock on C3: cold encode, 16 warm-up sweeps, then 8 profiled sweeps."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1903_07441_b200 import Planner, relax_cfg, warp_cfg
from scenes import scene_c3
T = int(sys.argv[1]) if len(sys.argv) > 1 else 4
rows = int(sys.argv[2]) if len(sys.argv) > 2 else 0
sc = scene_c3(0)
pl = Planner(sc.W, sc.H, 1, sc.cell_size, sc.origin, 0, torch.cuda.current_stream().cuda_stream)
pl.set_static(sc.static)
pl.set_obstacles(0, sc.robot, sc.goal, sc.tracks, warp_cfg(), warm=0)
pl.relax(relax_cfg(max_sweeps=4 * T, temporal_depth=T, rows_per_warp=rows))
pl.relax(relax_cfg(max_sweeps=2 * T, temporal_depth=T, rows_per_warp=rows))
torch.cuda.synchronize()
print("ok")
