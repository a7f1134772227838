"""Small workload for compute-sanitizer (tests/test_gpu_sanitizer.py): smoke() (C1, rows a1-a9), a
warm plan loop on a small random scene (speculative walk from the second tick on, tracker f1), the
lexicographic (mode 2) and Jacobi (mode 1) relaxations, the per-cell band and a local slab group."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import __graft_entry__ as G
from paper_1903_07441_b200 import Planner, band_cfg, relax_cfg, tracker_cfg, warp_cfg
from paper_1903_07441_b200.slab import make_group
from scenes import advance_scene, scene_random

G.smoke()
st = torch.cuda.current_stream().cuda_stream
sc0 = scene_random("san", 96, 3, 5, 8)
pl = Planner(sc0.W, sc0.H, 1, sc0.cell_size, sc0.origin, 0, st)
pl.set_static(sc0.static)
wc, bc = warp_cfg(), band_cfg(20, 2000, 4000)
for tick in range(3):
    sc = advance_scene(sc0, tick)
    rc = relax_cfg(max_sweeps=4000 if tick == 0 else 50, warm_start=1)
    pl.plan_step(0, [sc.robot], [sc.goal], sc.tracks, [sc.n_tracks], wc, rc, bc)
det = np.asarray(sc0.tracks, np.float64).reshape(-1, 20)[:, :2].copy()
pl.track_update(0, det, [len(det)], wc, tracker_cfg())
pl.relax(relax_cfg(max_sweeps=7, mode=2))
pl.relax(relax_cfg(max_sweeps=5, mode=1, check_every=1, tol=1e-3))
pl.band_index(0, band_cfg(3, 2000, 8))
pl.index_matrix(0)
pl.warp_map(sc0.robot)
pl.close()
pls = make_group(sc0.W, sc0.H, 3, sc0.static, sc0.robot, sc0.goal, sc0.tracks, wc, 4, stream=st)
pls[0].relax(relax_cfg(max_sweeps=30, check_every=8, tol=1e-4))
for p in pls:
    p.close()
torch.cuda.synchronize()
print("sanitize workload ok")
