import sys, os, time
sys.path.insert(0, '/root/repo') if os.path.exists('/root/repo') else None
sys.path.insert(0, os.getcwd())
import torch, numpy as np
from paper_1903_07441_b200 import Planner, relax_cfg, warp_cfg, band_cfg
from scenes import scene_c3
sc = scene_c3(0)
st = torch.cuda.current_stream()
pl = Planner(sc.W, sc.H, 1, sc.cell_size, sc.origin, 0, st.cuda_stream)
pl.set_static(sc.static)
pl.set_obstacles(0, sc.robot, sc.goal, sc.tracks, warp_cfg(), warm=0)
for S in (6, 60, 100):
    pl.profile(1)
    pl.relax(relax_cfg(max_sweeps=S), want_result=False)
    print(S, pl.profile_read())
    pl.profile(0)
pl.profile(1)
for k in range(3):
    pl.plan_step(0, [sc.robot], [sc.goal], sc.tracks, [sc.n_tracks], warp_cfg(), relax_cfg(max_sweeps=100), band_cfg(50, 32768, 65536), want_paths=False)
    print("step", k, pl.profile_read())
